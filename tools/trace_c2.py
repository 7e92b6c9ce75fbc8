"""Per-op trace (TNQVM_TRACE=1, stderr) of the bench step: C2 (Sycamore-53 m=10, bench.py's
plan) evaluated by one tnqvm_amplitude_batch call over 8 bitstrings (diagnostics only)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("TNQVM_TRACE", "1")
import bench  # noqa: E402
from paper_2104_10523_b200 import tnqvm as T  # noqa: E402
from synth import circuits as C  # noqa: E402

nb = int(sys.argv[1]) if len(sys.argv) > 1 else 8
_, _, plan, _ = bench.make_plan(T, C)
print(plan.info(), file=sys.stderr)
ctx = T.Context(0)
rows = [list(C.random_bitstring(53, 1000 + i)) for i in range(nb)]
ctx.amplitude_batch(plan, rows)
ctx.amplitude_batch(plan, rows)
print(ctx.stats(), file=sys.stderr)
