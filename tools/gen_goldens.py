"""Write the oracle-only golden values the GPU parity tests compare against
(tests/golden/*.txt).  Calls ONLY oracle/ and synth/ -- never the CUDA path.

    python tools/gen_goldens.py c2      # C2: Sycamore-53 m=10 whole amplitudes via O3 (minutes)
    python tools/gen_goldens.py c3      # C3 shape: 2 slices of a small-budget m=14 plan, 64-vectors
    python tools/gen_goldens.py c5      # C5 shape: 2 slices of a small-budget noisy m=8 plan

C3 / C5 (SURVEY §8(c) "a subset of slices against O3"): the sliced wire NAMES of the
product's plan are read as data from tests/golden/{c3,c5}_sliced_wires.json (written by
tools/plan_data.py); O3 fixes the same wires of its own network to the slice's mixed-radix
digits (first sliced wire = MSB, DESIGN R12) and contracts in complex128.

C2 (BASELINE.json configs[1], SURVEY §8(c) pin "the whole amplitude (C2) against O3's full
contraction"): a(b) = <b|U|0^53> (Eq.(1)) for the circuit of bench.py
(synth.circuits.sycamore53(10, seed=0)), contracted by O3 in complex128 along its own
greedy order with its own memory sub-slicing (every sub-slice summed: exact).
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import einsum_net as tn  # noqa: E402
from synth import circuits as C  # noqa: E402


def c2():
    ops = C.sycamore53(10, 0)
    rows = [("zeros", [0] * 53), ("rand1000", list(C.random_bitstring(53, 1000)))]
    lines = ["# C2 golden: Sycamore-53 m=10 (synth.circuits.sycamore53(10, 0)), whole amplitudes a(b) = <b|U|0^53>",
             "# (Eq.(1), P:L166-171) by O3 (oracle/einsum_net.py, numpy complex128, own greedy order,",
             "# restarts=16, own memory sub-slicing cap 2^26 elements, all sub-slices summed).",
             "# Written by tools/gen_goldens.py c2 (oracle only).  Columns: name bits re im seconds"]
    for name, bits in rows:
        t0 = time.perf_counter()
        a = tn.amplitude(ops, bits, restarts=16, cap_elems=2 ** 26)
        dt = time.perf_counter() - t0
        lines.append(f"{name} {''.join(map(str, bits))} {a.real:.17e} {a.imag:.17e} {dt:.1f}")
        print(lines[-1], flush=True)
    with open(os.path.join(ROOT, "tests", "golden", "c2_amplitudes.txt"), "w") as f:
        f.write("\n".join(lines) + "\n")


def _slices(name, net, ids, restarts):
    import json
    import numpy as np
    d = json.load(open(os.path.join(ROOT, "tests", "golden", f"{name}_sliced_wires.json")))
    t0 = time.perf_counter()
    vals = tn.slice_values(net, d["sliced"], ids, restarts=restarts, cap_elems=2 ** 26)
    dt = time.perf_counter() - t0
    out = {"plan_sha256": d["plan_sha256"], "slice_ids": ids, "seconds": round(dt, 1),
           "values": [[[float(z.real), float(z.imag)] for z in np.atleast_1d(np.asarray(v)).reshape(-1)] for v in vals]}
    with open(os.path.join(ROOT, "tests", "golden", f"{name}_slices.json"), "w") as f:
        json.dump(out, f, indent=0)
    print(name, dt, flush=True)


C3_BITS_SEED, C5_BITS_SEED = 1004, 1005


def c3():
    ops = C.sycamore53(14, 0)
    bits = list(C.random_bitstring(53, C3_BITS_SEED))
    for q in range(6):
        bits[q] = -1
    n = json.load(open(os.path.join(ROOT, "tests", "golden", "c3_sliced_wires.json")))["n_slices"]
    _slices("c3", tn.ket_network(ops, bits), [5 % n, (3 * n // 4 + 1) % n], restarts=16)


def c5():
    ops = C.noisy_grid_circuit(4, 5, 8, 0)
    bits = list(C.random_bitstring(20, C5_BITS_SEED))
    _slices("c5", tn.doubled_network(ops, ("project", bits)), [3, 2900], restarts=16)


if __name__ == "__main__":
    {"c2": c2, "c3": c3, "c5": c5}[sys.argv[1]]()
