"""C5 (20-qubit noisy grid, m=8, complex128) plan selection with tnqvm_plan_autotune over 16
planner seeds (diagnostics; prints the per-seed times and the winner)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2104_10523_b200 import tnqvm as T  # noqa: E402
from synth import circuits as C  # noqa: E402

ctx = T.Context(0)
circ = T.Circuit.from_oplist(C.noisy_grid_circuit(4, 5, 8, 0))
rows = [list(C.random_bitstring(20, 2000))]
seeds = list(range(16))
plan, ms = ctx.autotune_plan(circ, 16 << 31, seeds, rows, reps=2, dtype=T.C128, restarts=64)
best = seeds[min(range(len(seeds)), key=lambda i: ms[i])]
print(json.dumps({"config": "c5_noisy20_m8_c128", "ms_per_seed": {s: round(m, 2) for s, m in zip(seeds, ms)},
                  "best_seed": best, "best_ms": round(min(ms), 2), "log2_macs": plan.info()["log2_macs_sliced"]}))
