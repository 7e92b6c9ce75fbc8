#!/bin/bash
# intra-slice two-stream DAG: parity (full GPU suite), then C2 bench at 8 lanes and at 1 lane (per-slice latency proxy)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_dag.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_dag.log
grep -q "rc=0" gpurun_out/pytest_dag.log || exit 0
for v in 0 1; do for l in 8 1 2; do
  TNQVM_DAG=$v TNQVM_LANES=$l timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('dag', $v, 'lanes', $l, round(d['value'],1), round(d['ms_per_step'],3))" >> gpurun_out/dag.txt
done; done
echo done
