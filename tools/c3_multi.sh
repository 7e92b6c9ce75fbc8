#!/bin/bash
# C3 full on 1, 2 and 4 GPUs with one planner seed (gpurun --gpus 4); bit-identity checked after.
cd "$(dirname "$0")/.."
TAG=${TAG:-c3}
SEED=${SEED:-0}
P=29717
mkdir -p gpurun_out
rm -f gpurun_out/c3_amps_N*.npy
timeout 1500 python tools/bench_c3.py full --seed $SEED --restarts ${RESTARTS:-256} > gpurun_out/${TAG}_c3_full_N1.json 2> gpurun_out/${TAG}_c3_N1.err
for N in 2 4; do
  timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((P+N)) \
     tools/bench_c3.py full --gpus $N --seed $SEED --restarts ${RESTARTS:-256} > gpurun_out/${TAG}_c3_full_N$N.json 2> gpurun_out/${TAG}_c3_N$N.err
done
python - <<'PY'
import numpy as np, os
a = {n: np.load(f"gpurun_out/c3_amps_N{n}.npy") for n in (1, 2, 4) if os.path.exists(f"gpurun_out/c3_amps_N{n}.npy")}
print("c3 amps present:", sorted(a), "bit-identical:", all(np.array_equal(a[n], a[min(a)]) for n in a))
PY
