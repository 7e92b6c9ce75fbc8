#!/bin/bash
# tensor-core split-K (ystream) for huge-K tiny-output steps: parity, then C2 bench and C3 slice time with TNQVM_TC_SPLITK=0/1
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for v in 0 1; do
  TNQVM_TC_SPLITK=$v timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench_sk$v.json 2> gpurun_out/bench_sk$v.err
  TNQVM_TC_SPLITK=$v timeout 300 python tools/bench_c3.py probe --budget-log2 31 --slices 3 > gpurun_out/c3_probe_sk$v.json 2>&1
done
TNQVM_TRACE=1 TNQVM_GRAPH=0 timeout 300 python tools/bench_c3.py probe --budget-log2 31 --slices 2 > gpurun_out/c3_trace3.log 2>&1
TNQVM_TRACE=1 TNQVM_GRAPH=0 TNQVM_LANES=1 timeout 300 python tools/trace_c2.py 8 10 > gpurun_out/trace_c2b.log 2>&1
echo done
