# Bench every config (N=1) + PCIe probe. Outputs under gpurun_out/.
mkdir -p gpurun_out
python scripts/pcie_probe.py > gpurun_out/pcie.txt 2>&1
for c in c0 c1 c2 c3 c4 c4i; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  echo "$c rc=$?"
done
timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/bench_ref_c1.json 2> gpurun_out/bench_ref_c1.err
echo "ref rc=$?"
