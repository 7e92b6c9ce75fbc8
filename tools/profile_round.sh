#!/bin/bash
# GPU-box side: the whole round-evidence pass in one call.
#   1. pytest -m gpu            -> gpurun_out/pytest_gpu.log
#   2. default bench line       -> gpurun_out/bench.json (+ smoke)
#   3. ncu launch list of a short bench (only after the same command exited 0 without ncu)
#   4. per-launch DRAM traffic of every launch of the dominant kernel in one step
#   5. one `ncu --set full` capture of two launches of the dominant kernel
# usage: tools/profile_round.sh [kernel-regex] [skip-pytest]
K=${1:-tc_gemm_kernel}
mkdir -p gpurun_out
if [ -z "$2" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
  echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
fi
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
# ncu cannot replay the tcgen05 kernel node of a captured graph: profiled runs use TNQVM_GRAPH=0 (same kernels)
TNQVM_GRAPH=0 timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/plain.log 2>&1 && \
TNQVM_GRAPH=0 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_list.log 2>&1
TNQVM_GRAPH=0 timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
    --clock-control none --csv -k regex:$K -c 80 --log-file gpurun_out/traffic.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_traffic.log 2>&1
TNQVM_GRAPH=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 20 -c 2 \
    -o gpurun_out/prof_full python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
echo done
