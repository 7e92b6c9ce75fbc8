TNQVM_TRACE=1 TNQVM_GRAPH=0 timeout 300 python tools/bench_c3.py probe --budget-log2 31 --slices 2 > gpurun_out/c3_trace.log 2>&1
for ns in 1 2; do echo "== NSTG=$ns" >> gpurun_out/tc_sweep.log; TNQVM_TC_NSTG=$ns timeout 300 python tools/tc_probe.py 131072,128,128 131072,128,64 262144,32,64 262144,32,32 131072,32,64 65536,64,64 2048,32,2048 16384,32,128 16777216,64,16 16777216,32,64 >> gpurun_out/tc_sweep.log 2>&1; done
echo "== FLUSH_BN=128" >> gpurun_out/tc_sweep.log; TNQVM_TC_FLUSH_BN=128 timeout 300 python tools/tc_probe.py 131072,128,128 131072,128,64 4096,4096,4096 >> gpurun_out/tc_sweep.log 2>&1
echo "== GROUP=4" >> gpurun_out/tc_sweep.log; TNQVM_TC_GROUP=4 timeout 300 python tools/tc_probe.py 131072,128,128 131072,128,64 4096,4096,4096 >> gpurun_out/tc_sweep.log 2>&1
