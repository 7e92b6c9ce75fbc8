#!/bin/bash
# fused small-tensor CTA width: per-op C2 trace (1 lane), then C2 bench and C4 (expectation) at 256/512/1024 threads
mkdir -p gpurun_out
timeout 300 python tools/trace_c2.py 8 > /dev/null 2> gpurun_out/trace_c2_nt256.log
TNQVM_SMALL_NT=1024 timeout 300 python tools/trace_c2.py 8 > /dev/null 2> gpurun_out/trace_c2_nt1024.log
for nt in 256 512 1024; do
  TNQVM_SMALL_NT=$nt timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('nt', $nt, round(d['value'],1), round(d['ms_per_step'],3), round(d['e2e']['value'],1), d['roofline']['breakdown']['small'])" >> gpurun_out/small_nt.txt
  TNQVM_SMALL_NT=$nt timeout 300 python tools/bench_configs.py c4 c1 >> gpurun_out/small_nt_cfg_$nt.jsonl 2>&1
done
TNQVM_SMALL_NT=1024 timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_nt1024.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_nt1024.log
echo done
