cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests/test_gpu_parity.py -q --timeout=300 -k "gemm or c3 or c2 or batched" 2>&1 | tail -2
TNQVM_GRAPH=0 python tools/trace_c3.py 4 > gpurun_out/r02s_trace_c3.log 2>&1; grep "ms total" gpurun_out/r02s_trace_c3.log
grep -E "op45|op40 |op31 " gpurun_out/r02s_trace_c3.log | tail -3
timeout 900 python tools/bench_c3.py full > gpurun_out/r02s_c3_full_N1.json 2> gpurun_out/r02s_c3.err; grep -v NCCL gpurun_out/r02s_c3_full_N1.json | cut -c1-500
