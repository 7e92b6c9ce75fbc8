#!/bin/bash
# N = 2 (or 4) GPUs: multi-GPU parity test, then bench.py under torchrun (value, e2e through the batch call)
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
timeout 600 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/pytest_multi_N$N.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_multi_N$N.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 \
    bench.py --gpus $N --steps 100 --warmup 5 > gpurun_out/bench_N$N.json 2> gpurun_out/bench_N$N.err
echo done
