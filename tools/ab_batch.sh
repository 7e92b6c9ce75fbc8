#!/bin/bash
# amplitude_batch: new parity test first, then the full GPU suite, then bench (e2e through the batch call)
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "amplitude_batch or graph_replay" > gpurun_out/pytest_batch.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_batch.log
grep -q "rc=0" gpurun_out/pytest_batch.log || exit 0
timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/bench_batch.json 2> gpurun_out/bench_batch.err
for b in 1 4 25; do
  E2E_BATCH=$b timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('batch', $b, round(d['value'],1), round(d['e2e']['value'],1), d['e2e']['single_call_value'])" >> gpurun_out/batch_sweep.txt
done
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_all.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_all.log
echo done
