"""Measured throughput of the C2 bench step (8 single-amplitude bitstrings per
tnqvm_amplitude_batch call) for several planner seeds (diagnostics: plans with equal
predicted cost differ in measured time).  usage: python tools/seed_sweep.py s0 s1 ..."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2104_10523_b200 import tnqvm as T  # noqa: E402
from synth import circuits as C  # noqa: E402

ctx = T.Context(0)
rows = [list(C.random_bitstring(53, 1000 + i)) for i in range(8)]
circ = T.Circuit.from_oplist(C.sycamore53(bench.CYCLES, bench.CIRCUIT_SEED))
for s in [int(a) for a in sys.argv[1:]]:
    t0 = time.perf_counter()
    plan = T.Plan(circ, [], bench.BUDGET_BYTES, seed=s, restarts=bench.RESTARTS, dtype=T.C64,
                  min_slices=bench.MIN_SLICES, cost_model=int(os.environ.get("COST_MODEL", "1")),
                  partition=int(os.environ.get("PARTITION", "1")))
    tp = time.perf_counter() - t0
    for _ in range(3):
        ctx.amplitude_batch(plan, rows)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(15):
        ctx.amplitude_batch(plan, rows)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 15
    info = plan.info()
    print(json.dumps({"seed": s, "amps_per_s": round(8e3 / ms, 1), "ms_per_call": round(ms, 3), "plan_s": round(tp, 1),
                      "log2_macs": round(info["log2_macs_sliced"], 4), "log2_max": info["log2_max_intermediate"],
                      "n_steps": info["n_steps"], "bytes": info["bytes_sliced"]}), flush=True)
    del plan
