#!/bin/bash
# End-of-round multi-GPU pass (gpurun --gpus 4): C3 full on 1, 2 and 4 GPUs (bit-identity of the
# 64 amplitudes), C2 bench at 2 and 4 GPUs, the multi-rank pytest, and the C1/C4/C5 configs.
cd "$(dirname "$0")/.."
TAG=${TAG:-final}
P=29617
mkdir -p gpurun_out
timeout 900 python tools/bench_c3.py full > gpurun_out/${TAG}_c3_full_N1.json 2> gpurun_out/${TAG}_c3_N1.err
for N in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((P+10+N)) \
     tools/bench_c3.py full --gpus $N > gpurun_out/${TAG}_c3_full_N$N.json 2> gpurun_out/${TAG}_c3_N$N.err
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((P+N)) \
     bench.py --gpus $N --steps 20 --warmup 5 > gpurun_out/${TAG}_bench_N$N.json 2> gpurun_out/${TAG}_bench_N$N.err
done
timeout 900 python -m pytest tests/test_gpu_multi.py -q --timeout=600 > gpurun_out/${TAG}_pytest_multi.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest_multi.log
timeout 900 python tools/bench_configs.py c1 c4 c5 > gpurun_out/${TAG}_configs.jsonl 2> gpurun_out/${TAG}_configs.err
python - <<'PY'
import numpy as np, os
a = {n: np.load(f"gpurun_out/c3_amps_N{n}.npy") for n in (1, 2, 4) if os.path.exists(f"gpurun_out/c3_amps_N{n}.npy")}
print("c3 amps present:", sorted(a), "bit-identical:", all(np.array_equal(a[n], a[min(a)]) for n in a))
PY
tail -2 gpurun_out/${TAG}_pytest_multi.log
echo done
