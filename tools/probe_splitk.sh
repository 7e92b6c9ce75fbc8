#!/bin/bash
# split-K tail of C2 (the last step of every slice): one --set full capture, plus the C2 plan's slice count sweep at N=1
mkdir -p gpurun_out
TNQVM_GRAPH=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:splitk_big_kernel -s 4 -c 1 \
    -o gpurun_out/prof_splitk python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_splitk.log 2>&1
for s in 1 2 4 16; do
  BENCH_MIN_SLICES=$s timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('min_slices', $s, d['config']['n_slices'], round(d['value'],1), round(d['e2e']['value'],1))" >> gpurun_out/slices_sweep.txt
done
echo done
