cd "$(dirname "$0")/.."
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "permute or c2 or batched" --timeout=300 2>&1 | tail -2
TNQVM_TRACE=1 TNQVM_GRAPH=0 python tools/trace_c2.py 8 2>&1 | grep -E "permute|ms total" | tail -3
python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | cut -c1-170
timeout 600 python tools/kernel_bench.py n1 > gpurun_out/r02p_n1.jsonl 2>&1; tail -4 gpurun_out/r02p_n1.jsonl | cut -c1-200
