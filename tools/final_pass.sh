#!/bin/bash
# Round-end evidence with the final code: lane sweep, default bench line (with cpu_baseline),
# ncu launch list, per-launch DRAM traffic of the dominant kernel, one --set full capture.
mkdir -p gpurun_out
for l in 2 3 4 6; do TNQVM_LANES=$l timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench_lanes$l.json 2>/dev/null; done
bash tools/profile_round.sh tc_gemm_kernel skip
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo done
