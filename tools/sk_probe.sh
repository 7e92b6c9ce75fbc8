cd "$(dirname "$0")/.."
TNQVM_TRACE=1 TNQVM_GRAPH=0 python tools/trace_c2.py 8 > gpurun_out/r02n_trace.log 2>&1
TNQVM_SPLITK_BLOCKED_EXPERIMENT=1 TNQVM_TRACE=1 TNQVM_GRAPH=0 python tools/trace_c2.py 8 > gpurun_out/r02n_trace_blk.log 2>&1
python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | cut -c1-170
TNQVM_SPLITK_BLOCKED_EXPERIMENT=1 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | cut -c1-170
grep -E "splitk|permute" gpurun_out/r02n_trace.log | tail -4; grep -E "splitk|permute" gpurun_out/r02n_trace_blk.log | tail -4
