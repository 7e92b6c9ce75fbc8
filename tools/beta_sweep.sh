#!/bin/bash
# planner time-model beta sweep (R18): C5 (c128 noisy) and C2 (bench, c64)
for b in 20 40; do echo "c5 beta=$b"; TNQVM_PLAN_BETA=$b timeout 600 python tools/bench_configs.py c5 2>&1 | cut -c1-200; done
for b in 12 48; do echo "c2 beta=$b"; TNQVM_PLAN_BETA=$b python bench.py --no-cpu-baseline --steps 50 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['config']['log2_macs'])"; done
