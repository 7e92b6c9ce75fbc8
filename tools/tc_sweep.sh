#!/bin/bash
# tcgen05 GEMM parameter sweep on representative C2 shapes (tc_probe timing, CUDA events)
S="131072,128,128 131072,128,64 262144,32,64 262144,32,32 1048576,16,32 65536,64,64"
for cfg in "256 2" "128 2" "256 1" "128 1" "64 1"; do
  set -- $cfg
  echo "== BN<=$1 NSTG=$2"
  TNQVM_TC_BN=$1 TNQVM_TC_NSTG=$2 python tools/tc_probe.py $S 2>&1 | grep "method=2"
done
