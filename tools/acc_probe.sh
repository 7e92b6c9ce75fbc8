cd $GRAFT_REPO_ROOT
for g in 0 1 2 4; do TNQVM_TC_GROUP_EXPERIMENT=$g python tools/tc_accuracy.py; done > gpurun_out/r02b_tc_accuracy.jsonl 2> gpurun_out/r02b_tc_accuracy.err
TNQVM_TRACE=1 TNQVM_GRAPH=0 python tools/trace_c2.py 8 > gpurun_out/r02b_trace_c2.log 2>&1
tail -2 gpurun_out/r02b_tc_accuracy.err
