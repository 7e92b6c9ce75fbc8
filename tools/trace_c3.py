"""Per-op trace (TNQVM_TRACE=1, stderr) of C3: Sycamore-53 m=14, open qubits 0..5, 2^31-element
budget (tools/bench_c3.py's plan), evaluated on `n` slices batched into one unit set."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("TNQVM_TRACE", "1")
from paper_2104_10523_b200 import tnqvm as T  # noqa: E402
from synth import circuits as C  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4
ops = C.sycamore53(14, 0)
plan = T.Plan(T.Circuit.from_oplist(ops), list(range(6)), 8 << 31, seed=int(os.environ.get("C3_SEED", "2")),
              restarts=int(os.environ.get("C3_RESTARTS", "4096")), dtype=T.C64)
print(plan.info(), file=sys.stderr)
ctx = T.Context(0)
bits = list(C.random_bitstring(53, 3000))
for q in range(6):
    bits[q] = -1
ctx.eval_slices(plan, bits, list(range(n)))
ctx.eval_slices(plan, bits, list(range(n)))
print(ctx.stats(), file=sys.stderr)
