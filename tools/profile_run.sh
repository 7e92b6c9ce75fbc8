#!/bin/bash
# GPU-box side, call 1: the default bench line, then the ncu launch list of a short bench
# (one ncu per call; the launch list only after the same command exited 0 without ncu).
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv > gpurun_out/smi_before.csv
# (ncu cannot replay the tcgen05 kernel node of a captured graph: the profiled runs use TNQVM_GRAPH=0, same kernels)
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
TNQVM_GRAPH=0 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/plain.log 2>&1 && \
TNQVM_GRAPH=0 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_list.log 2>&1
echo done
