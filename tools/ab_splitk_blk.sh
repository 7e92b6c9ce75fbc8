#!/bin/bash
# split-K register blocking for complex64 (TNQVM_SPLITK_BLOCKED): parity with it on, C2 bench A/B
mkdir -p gpurun_out
TNQVM_SPLITK_BLOCKED=1 timeout 600 python -m pytest tests -m gpu -x -q -k "splitk or c2_bench or sycamore or sliced or lanes" > gpurun_out/pytest_blk.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_blk.log
grep -q "rc=0" gpurun_out/pytest_blk.log || exit 0
for x in 1 0 1 0; do TNQVM_SPLITK_BLOCKED=$x timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('blocked', $x, round(d['value'],1), round(d['e2e']['value'],1), d['roofline']['breakdown']['splitk'])" >> gpurun_out/blk_bench.txt; done
echo done
