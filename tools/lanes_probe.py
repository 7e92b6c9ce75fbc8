"""Per-step device time of the C2 bench step over many steps for a given TNQVM_LANES."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2104_10523_b200 import tnqvm as T  # noqa: E402
from synth import circuits as C  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 40
ops = C.sycamore53(10, 0)
plan = T.Plan(T.Circuit.from_oplist(ops), [], 16 << 30, seed=0, restarts=256, dtype=T.C64, min_slices=8)
ctx = T.Context(0, stream=torch.cuda.current_stream().cuda_stream)
bits = [[0] * 53] + [list(C.random_bitstring(53, 1000 + i)) for i in range(4)]
out = []
for i in range(steps):
    t = time.perf_counter()
    a = ctx.amplitude(plan, bits[i % 5])
    w = time.perf_counter() - t
    s = ctx.stats()
    free, tot = torch.cuda.mem_get_info()
    out.append(f"{i} dev={s['ms_total']:.2f}ms wall={w * 1e3:.2f}ms host={s['host_ms']:.2f}ms graph={s['graph']} free={free / 2**30:.1f}G "
               f"alloc={torch.cuda.memory_allocated() / 2**30:.2f}G reserved={torch.cuda.memory_reserved() / 2**30:.2f}G a={a}")
print("\n".join(out))
