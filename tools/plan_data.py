"""Write the plan DATA the oracle's slice-subset goldens need (host planner only, no GPU):
the sliced wire names {side, qubit, segment} of a plan, in slice-digit order (P:L134
slicing; R7 wire naming, R12 enumeration).  The oracle reads them as data to
fix the same wires of its OWN network (oracle/einsum_net.py slice_values).

    python tools/plan_data.py c3    # -> tests/golden/c3_sliced_wires.json
    python tools/plan_data.py c5    # -> tests/golden/c5_sliced_wires.json
    python tools/plan_data.py c2    # -> tests/golden/c2_sliced_wires.json (bench.py's plan; read by
                                    #    bench.py --impl reference, which never loads libtnqvm)
"""
import hashlib
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2104_10523_b200 import tnqvm as T  # noqa: E402
from synth import circuits as C  # noqa: E402

# C3 shape (Sycamore-53 m=14, open qubits 0..5) planned at a small budget so that one slice
# is ~2^30 complex MACs on the GPU plan (the throughput plan's slices are 2^40)
C3 = dict(cycles=14, seed=0, open=list(range(6)), budget=8 << 22, restarts=64, plan_seed=0, dtype="c64")
# C5 shape (4x5 noisy grid m=8, doubled network, complex128) at a small budget
C5 = dict(rows=4, cols=5, cycles=8, seed=0, open=[], budget=16 << 20, restarts=32, plan_seed=0, dtype="c128")


# C2: bench.py's plan (Sycamore-53 m=10, 16 GiB budget, 4096 restarts, planner seed 2, min_slices 8,
# time-model cost)
C2 = dict(cycles=10, seed=0, open=[], budget=16 << 30, restarts=4096, plan_seed=2, dtype="c64", min_slices=8,
          cost_model=1)


def c2_plan():
    ops = C.sycamore53(C2["cycles"], C2["seed"])
    return ops, T.Plan(T.Circuit.from_oplist(ops), C2["open"], C2["budget"], restarts=C2["restarts"],
                       seed=C2["plan_seed"], dtype=T.C64, min_slices=C2["min_slices"], cost_model=C2["cost_model"])


def c3_plan():
    ops = C.sycamore53(C3["cycles"], C3["seed"])
    return ops, T.Plan(T.Circuit.from_oplist(ops), C3["open"], C3["budget"], restarts=C3["restarts"],
                       seed=C3["plan_seed"], dtype=T.C64)


def c5_plan():
    ops = C.noisy_grid_circuit(C5["rows"], C5["cols"], C5["cycles"], C5["seed"])
    return ops, T.Plan(T.Circuit.from_oplist(ops), C5["open"], C5["budget"], restarts=C5["restarts"],
                       seed=C5["plan_seed"], dtype=T.C128)


def write(name, cfg, plan):
    d = dict(cfg)
    d["sliced"] = plan.sliced_wires()
    d["n_slices"] = plan.info()["n_slices"]
    d["log2_macs_sliced"] = plan.info()["log2_macs_sliced"]
    d["plan_sha256"] = hashlib.sha256(plan.json().encode()).hexdigest()
    with open(os.path.join(ROOT, "tests", "golden", f"{name}_sliced_wires.json"), "w") as f:
        json.dump(d, f, indent=1, sort_keys=True)
    print(name, d["n_slices"], d["log2_macs_sliced"])


if __name__ == "__main__":
    name = sys.argv[1]
    cfg, fn = {"c2": (C2, c2_plan), "c3": (C3, c3_plan), "c5": (C5, c5_plan)}[name]
    write(name, cfg, fn()[1])
