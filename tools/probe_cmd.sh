python tools/lanes_probe.py 150 > gpurun_out/lanes.log 2>&1
(for i in $(seq 1 30); do nvidia-smi --query-gpu=clocks.sm,power.draw,temperature.gpu,clocks_event_reasons.active --format=csv,noheader; sleep 0.1; done) > gpurun_out/smi.log 2>&1 &
TNQVM_GRAPH=0 python tools/lanes_probe.py 150 > gpurun_out/lanes_nog.log 2>&1
wait
