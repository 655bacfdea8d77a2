#!/bin/bash
# Code-path check of bench.py at N=2 (torchrun, two ranks sharing the one GPU
# of this box): IPC halo default, NCCL halo, both arms. Numbers meaningless.
mkdir -p gpurun_out
export U16M_BENCH_SHARE_GPU=1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517"
timeout 900 $TR bench.py --gpus 2 --steps 3 --warmup 3 --config c1 > gpurun_out/dist_c1_ipc.json 2> gpurun_out/dist_c1_ipc.err; echo "ipc rc=$?"
# (the NCCL halo needs distinct GPUs: covered by tests/test_gpu_dist.py)
# timeout 900 $TR bench.py --gpus 2 --steps 3 --warmup 3 --config c1 --halo nccl > gpurun_out/dist_c1_nccl.json 2> gpurun_out/dist_c1_nccl.err; echo "nccl rc=$?"
timeout 900 $TR bench.py --gpus 2 --steps 3 --warmup 3 --impl reference --config c1 > gpurun_out/dist_c1_ref.json 2> gpurun_out/dist_c1_ref.err; echo "ref rc=$?"
timeout 1200 $TR bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/dist_c4.json 2> gpurun_out/dist_c4.err; echo "c4 rc=$?"
