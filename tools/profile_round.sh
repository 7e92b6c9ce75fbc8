#!/bin/bash
# GPU-box side: the round-evidence pass in one call (logs -> gpurun_out/<TAG>_*).
#   1. pytest -m gpu + smoke (skip with SKIP_TESTS=1)
#   2. default bench line (with the CPU baseline)
#   3. ncu launch list of a short bench (after the same command exited 0 without ncu)
#   4. per-launch DRAM traffic of the GEMM launches of one timed step (N=1: CPS chunks)
#   5. `ncu --set full` of the first chunk of that step: its TCPC tcgen05 GEMMs, split-K and permutes
# (launch counts: bench.py runs 3 warm-up batch calls (CPS chunks each) and 2 single calls (1
# chunk each) before the timed step; TCPC = tcgen05 launches per chunk, XPC = the split-K and
# permute launches per chunk, of the bench plan; CPS = chunks per step, 1 at 64 units per chunk)
# usage: TAG=r02c tools/profile_round.sh
cd "$(dirname "$0")/.."
TAG=${TAG:-prof}
TCPC=${TCPC:-10}
XPC=${XPC:-2}
CPS=${CPS:-1}
PRE=$((3 * CPS + 2))
mkdir -p gpurun_out
if [ -z "$SKIP_TESTS" ]; then
  timeout 1500 python -m pytest tests -m gpu -q --timeout=400 > gpurun_out/${TAG}_pytest.log 2>&1
  echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
  echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
fi
timeout 600 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
# profiled runs launch directly (TNQVM_GRAPH=0): the same kernels, ncu replays them one by one
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
TNQVM_GRAPH=0 timeout 300 $B > gpurun_out/${TAG}_plain.log 2>&1 && \
TNQVM_GRAPH=0 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${TAG}_launches.csv $B > gpurun_out/${TAG}_ncu_list.log 2>&1
TNQVM_GRAPH=0 timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
    --clock-control none --csv -k regex:tc_gemm -s $((PRE * TCPC)) -c $((CPS * TCPC)) --log-file gpurun_out/${TAG}_traffic.csv \
    $B > gpurun_out/${TAG}_ncu_traffic.log 2>&1
TNQVM_GRAPH=0 timeout 1200 ncu --set full --clock-control none --import-source on \
    -k regex:'tc_gemm|splitk_big_kernel|splitk_lane|permute' -s $((PRE * (TCPC + XPC))) -c $((TCPC + XPC)) -o gpurun_out/${TAG}_full $B > gpurun_out/${TAG}_ncu_full.log 2>&1
echo done
