#!/bin/bash
# CTA-pair tcgen05 GEMM: parity first (bounded), then kernel shapes / C2 bench / C3 slice with TNQVM_TC_CG=1/2
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "gemm_tcgen05" > gpurun_out/pytest_tc.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_tc.log
grep -q "pytest rc=0" gpurun_out/pytest_tc.log || exit 0
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for v in 1 2; do
  TNQVM_TC_CG=$v timeout 400 python tools/kernel_bench.py n2c 2>&1 | grep "^{" > gpurun_out/kb_n2c_cg$v.jsonl
  TNQVM_TC_CG=$v timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench_cg$v.json 2> gpurun_out/bench_cg$v.err
  TNQVM_TC_CG=$v timeout 300 python tools/bench_c3.py probe --budget-log2 31 --slices 3 > gpurun_out/c3_probe_cg$v.json 2>&1
done
echo done
