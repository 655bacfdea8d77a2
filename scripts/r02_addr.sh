mkdir -p gpurun_out
for c in "" "expandable_segments:True" "backend:cudaMallocAsync"; do
  PYTORCH_CUDA_ALLOC_CONF=$c python scripts/addr_range_probe.py >> gpurun_out/addr_range.txt 2>&1
done
