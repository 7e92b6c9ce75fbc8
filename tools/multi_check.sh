#!/bin/bash
# multi-GPU pass (run under gpurun --gpus 4): multi-rank pytest, C2 bench at 2 and 4 GPUs,
# C3 full at 2 and 4 GPUs (the same plan, bit-identity of the 64 amplitudes checked after).
cd "$(dirname "$0")/.."
TAG=${TAG:-multi}
P=29517
timeout 900 python -m pytest tests/test_gpu_multi.py -q --timeout=600 > gpurun_out/${TAG}_pytest_multi.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest_multi.log
for N in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((P+N)) \
     bench.py --gpus $N --steps 20 --warmup 5 > gpurun_out/${TAG}_bench_N$N.json 2> gpurun_out/${TAG}_bench_N$N.err
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((P+10+N)) \
     tools/bench_c3.py full --gpus $N > gpurun_out/${TAG}_c3_full_N$N.json 2> gpurun_out/${TAG}_c3_N$N.err
done
python - <<'PY'
import numpy as np, os
a = {n: np.load(f"gpurun_out/c3_amps_N{n}.npy") for n in (1, 2, 4) if os.path.exists(f"gpurun_out/c3_amps_N{n}.npy")}
print("c3 amps present:", sorted(a), "bit-identical:", all(np.array_equal(a[n], a[min(a)]) for n in a))
PY
tail -2 gpurun_out/${TAG}_pytest_multi.log; for N in 2 4; do cut -c1-200 gpurun_out/${TAG}_bench_N$N.json; cut -c1-420 gpurun_out/${TAG}_c3_full_N$N.json; done
