"""Per-op trace of one Sycamore-53 amplitude (bench config) -- TNQVM_TRACE=1 output on stderr."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("TNQVM_TRACE", "1")

from paper_2104_10523_b200 import tnqvm as T  # noqa: E402
from synth import circuits as C  # noqa: E402

min_slices = int(sys.argv[1]) if len(sys.argv) > 1 else 64
cycles = int(sys.argv[2]) if len(sys.argv) > 2 else 10
ops = C.sycamore53(cycles, 0)
circ = T.Circuit.from_oplist(ops)
plan = T.Plan(circ, [], 16 << 30, seed=0, restarts=256, dtype=T.C64, min_slices=min_slices)
print(plan.info(), file=sys.stderr)
ctx = T.Context(0)

a = ctx.amplitude(plan, [0] * 53)
t = time.perf_counter()
a = ctx.amplitude(plan, [0] * 53)
print("amp", a, "wall", time.perf_counter() - t, ctx.stats(), file=sys.stderr)
