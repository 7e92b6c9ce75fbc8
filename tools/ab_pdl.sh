#!/bin/bash
# A/B of programmatic dependent launch: parity tests, then the C2 bench and tiny tc shapes with TNQVM_PDL=0/1
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for pdl in 0 1; do
  TNQVM_PDL=$pdl timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench_pdl$pdl.json 2> gpurun_out/bench_pdl$pdl.err
  TNQVM_PDL=$pdl timeout 300 python tools/tc_probe.py 128,16,16 2048,32,32 16384,32,128 2048,32,2048 65536,64,64 262144,32,64 > gpurun_out/tc_pdl$pdl.log 2>&1
done
echo done
