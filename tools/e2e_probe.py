"""Where the e2e time of tnqvm_amplitude_batch goes: device span of each batch (ms_total),
host enqueue time (host_ms) and wall time per batch, for C2's bench plan."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2104_10523_b200 import tnqvm as T  # noqa: E402
from synth import circuits as C  # noqa: E402

ops, circ, plan, _ = bench.make_plan(T, C)
ctx = T.Context(0)
rows = [list(C.random_bitstring(53, 1000 + i)) for i in range(10)]
for nb in (10, 10, 10, 1, 1, 1):
    t = time.perf_counter()
    ctx.amplitude_batch(plan, rows[:nb])
    w = (time.perf_counter() - t) * 1e3
    st = ctx.stats()
    print(f"nb {nb} wall {w:.3f} ms  device span {st['ms_total']:.3f} ms  host enqueue {st['host_ms']:.3f} ms  "
          f"per amp: wall {w / nb:.3f} device {st['ms_total'] / nb:.3f}", file=sys.stderr)
t = time.perf_counter()
for r in rows:
    ctx.amplitude(plan, r)
print(f"10 single calls wall {(time.perf_counter() - t) * 1e3:.3f} ms", file=sys.stderr)
