#!/bin/bash
cd "$(dirname "$0")/.."
TAG=${TAG:-probe}
TNQVM_TC_DEBUG=1 python tools/tc_dbg.py > gpurun_out/${TAG}_dbg.log 2>&1
TAG=$TAG python tools/tc_accuracy.py > gpurun_out/${TAG}_tc.jsonl 2> gpurun_out/${TAG}_tc.err
timeout 900 python -m pytest tests/test_gpu_parity.py -q --timeout=400 -k "gemm or c2 or batched or sycamore" > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
TNQVM_TRACE=1 TNQVM_GRAPH=0 python tools/trace_c2.py 8 > gpurun_out/${TAG}_trace.log 2>&1
tail -2 gpurun_out/${TAG}_pytest.log; cut -c1-200 gpurun_out/${TAG}_bench.json
