#!/bin/bash
# full GPU tests + smoke + bench + C3 on 1 GPU (TAG names the outputs)
cd "$(dirname "$0")/.."
TAG=${TAG:-check}
timeout 1500 python -m pytest tests -m gpu -q --timeout=600 > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
timeout 600 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
timeout 900 python tools/bench_c3.py full > gpurun_out/${TAG}_c3_full_N1.json 2> gpurun_out/${TAG}_c3.err
tail -2 gpurun_out/${TAG}_pytest.log; tail -1 gpurun_out/${TAG}_smoke.log; cut -c1-300 gpurun_out/${TAG}_bench.json; cut -c1-600 gpurun_out/${TAG}_c3_full_N1.json; tail -3 gpurun_out/${TAG}_c3.err
