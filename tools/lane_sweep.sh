#!/bin/bash
for l in 1 2 3 4; do echo "lanes=$l $(TNQVM_LANES=$l python bench.py --no-cpu-baseline --steps 50 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"])')"; done
for ms in 16 32; do echo "min_slices=$ms $(BENCH_MIN_SLICES=$ms python bench.py --no-cpu-baseline --steps 50 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["config"]["log2_macs"], d["config"]["n_slices"])')"; done
for ms in 16 32; do echo "min_slices=$ms lanes=3 $(TNQVM_LANES=3 BENCH_MIN_SLICES=$ms python bench.py --no-cpu-baseline --steps 50 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"])')"; done
