#!/bin/bash
mkdir -p gpurun_out
for l in 8 6 10 12 16 8; do TNQVM_LANES=$l timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('lanes', $l, round(d['value'],1), round(d['e2e']['value'],1))" >> gpurun_out/lane_sweep2.txt; done
echo done
