#!/bin/bash
# N2 accuracy + timing probe, then the N2 parity tests and a short bench (TAG names the outputs)
cd "$(dirname "$0")/.."
TAG=${TAG:-probe}
TAG=$TAG python tools/tc_accuracy.py > gpurun_out/${TAG}_tc.jsonl 2> gpurun_out/${TAG}_tc.err
timeout 900 python -m pytest tests -m gpu -q --timeout=400 > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
TNQVM_TRACE=1 TNQVM_GRAPH=0 python tools/trace_c2.py 8 > gpurun_out/${TAG}_trace.log 2>&1
tail -2 gpurun_out/${TAG}_pytest.log; cut -c1-200 gpurun_out/${TAG}_bench.json
