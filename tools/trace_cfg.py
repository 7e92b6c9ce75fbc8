"""Per-op trace (TNQVM_TRACE=1) of one evaluation of a named config: c5 (noisy 20q m=8),
c4 (QAOA 40q p=2, first terms), c3 (Sycamore-53 m=14 + 6 open, a few slices)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("TNQVM_TRACE", "1")

from paper_2104_10523_b200 import tnqvm as T  # noqa: E402
from synth import circuits as C  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c5"
ctx = T.Context(0)
if cfg == "c5":
    m = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    ops = C.noisy_grid_circuit(4, 5, m, 0)
    p = T.Plan(T.Circuit.from_oplist(ops), [], 16 << 31, dtype=T.C128, restarts=64)
    print(p.info(), file=sys.stderr)
    t = time.perf_counter()
    v = ctx.amplitude(p, list(C.random_bitstring(20, 2000)))
    print("prob", v, "wall", time.perf_counter() - t, ctx.stats(), file=sys.stderr)
elif cfg == "c4":
    ops, terms = C.qaoa40(0)
    circ = T.Circuit.from_oplist(ops)
    t = time.perf_counter()
    tot = ctx.expectation(circ, terms[:4], dtype=T.C128, restarts=16)
    print("H4", tot, "wall", time.perf_counter() - t, ctx.stats(), file=sys.stderr)
elif cfg == "c3":
    ops = C.sycamore53(14, 0)
    p = T.Plan(T.Circuit.from_oplist(ops), list(range(6)), 8 << 32, restarts=64)
    print(p.info(), file=sys.stderr)
    bits = list(C.random_bitstring(53, 3000))
    for q in range(6):
        bits[q] = -1
    t = time.perf_counter()
    ctx.eval_slices(p, bits, [0, 1])
    print("wall", time.perf_counter() - t, ctx.stats(), file=sys.stderr)
