cd "$(dirname "$0")/.."
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "permute or batched" --timeout=300 2>&1 | tail -1
TNQVM_TRACE=1 TNQVM_GRAPH=0 python tools/trace_c2.py 8 2>&1 | grep -E "permute|ms total" | tail -3
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
TNQVM_GRAPH=0 $B > /dev/null 2>&1 && TNQVM_GRAPH=0 timeout 600 ncu --metrics gpu__time_duration.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:permute -c 2 $B 2>/dev/null | grep -E "permute" | cut -c1-300 | tail -10
