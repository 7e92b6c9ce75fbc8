cd "$(dirname "$0")/.."
TNQVM_TRACE=1 TNQVM_GRAPH=0 python tools/trace_c2.py 8 2>&1 | grep -A40 "ms total" | tail -30 > gpurun_out/r02q_gather.log
TNQVM_NO_GATHER_EXPERIMENT=1 TNQVM_TRACE=1 TNQVM_GRAPH=0 python tools/trace_c2.py 8 2>&1 | grep -A40 "ms total" | tail -34 > gpurun_out/r02q_nogather.log
