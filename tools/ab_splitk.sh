#!/bin/bash
# split-K vectorised X gather: kernel parity, C2 bench A/B (TNQVM_SPLITK_XVEC), one ncu capture of the split-K kernel
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "splitk or c2_bench or sycamore or sliced or lanes" > gpurun_out/pytest_sk.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_sk.log
grep -q "rc=0" gpurun_out/pytest_sk.log || exit 0
for x in 1 0 1; do TNQVM_SPLITK_XVEC=$x timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('xvec', $x, round(d['value'],1), round(d['e2e']['value'],1), d['roofline']['breakdown']['splitk'])" >> gpurun_out/sk_bench3.txt; done
TNQVM_GRAPH=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:splitk_big_kernel -s 4 -c 1 \
    -o gpurun_out/prof_splitk3 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_splitk3.log 2>&1
echo done
