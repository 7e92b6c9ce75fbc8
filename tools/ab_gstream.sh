#!/bin/bash
# graph launched on ctx.stream vs on gstream with an event pair: full GPU suite, bench A/B
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gs.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gs.log
grep -q "rc=0" gpurun_out/pytest_gs.log || exit 0
for g in 0 1 0 1; do TNQVM_GRAPH_GSTREAM=$g timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('gstream', $g, round(d['value'],1), round(d['e2e']['value'],1), round(d['e2e']['single_call_value'],1))" >> gpurun_out/gs_ab.txt; done
echo done
