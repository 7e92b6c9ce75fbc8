#!/bin/bash
# on-chip W split + streamed-Y split-K: parity, kernel shapes (TNQVM_TC_WSPLIT=0/1), C2 bench, C3 slice trace
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "gemm or sycamore or sliced or graph" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for w in 0 1; do TNQVM_TC_WSPLIT=$w timeout 400 python tools/kernel_bench.py n2c 2>&1 | grep "^{" > gpurun_out/kb_n2c_w$w.jsonl; done
for w in 0 1; do TNQVM_TC_WSPLIT=$w timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench_w$w.json 2> gpurun_out/bench_w$w.err; done
TNQVM_TRACE=1 TNQVM_GRAPH=0 timeout 300 python tools/bench_c3.py probe --budget-log2 31 --slices 2 > gpurun_out/c3_trace2.log 2>&1
timeout 300 python tools/bench_c3.py probe --budget-log2 31 --slices 3 > gpurun_out/c3_probe2.json 2>&1
echo done
