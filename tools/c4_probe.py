"""Per-call wall / device time of the C4 QAOA expectation (both dtypes, graphs on/off)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2104_10523_b200 import tnqvm as T  # noqa: E402
from synth import circuits as C  # noqa: E402

ops, terms = C.qaoa40(0)
circ = T.Circuit.from_oplist(ops)
ctx = T.Context(0)
for dtype in (T.C128, T.C64):
    out = []
    for i in range(8):
        t = time.perf_counter()
        ctx.expectation(circ, terms, dtype=dtype, restarts=16)
        out.append(f"{(time.perf_counter() - t) * 1e3:.1f}/{ctx.stats()['ms_total']:.1f}")
    print("c128" if dtype == T.C128 else "c64", os.environ.get("TNQVM_GRAPH", "1"), " ".join(out), flush=True)
