#!/bin/bash
# GPU-box side, call 2: one `ncu --set full` capture of kernel $1 (regex) inside the bench step.
K=${1:-tc_gemm_kernel}
S=${2:-20}
TNQVM_GRAPH=0 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/plain_full.log 2>&1 && \
TNQVM_GRAPH=0 ncu --set full --clock-control none --import-source on -k regex:$K -s $S -c 2 \
    -o gpurun_out/prof_full python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
echo done
