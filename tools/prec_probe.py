"""c64 vs c128 vs O3 per-slice error on the Sycamore-53 m=8 test plan."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2104_10523_b200 import tnqvm as T
from synth import circuits as C
from oracle import einsum_net as tn
ops = C.sycamore53(8, seed=0)
c = T.Circuit.from_oplist(ops)
ctx = T.Context(0)
bits = C.random_bitstring(53, 1001)
p64 = T.Plan(c, [], 8 << 22, restarts=32, min_slices=16)
p128 = T.Plan(c, [], 16 << 22, restarts=32, min_slices=16, dtype=T.C128)
print("same sliced", p64.sliced_wires() == p128.sliced_wires(), p64.info())
ids = list(range(p64.info()["n_slices"]))
g64 = ctx.eval_slices(p64, bits, ids)[:, 0]
g128 = ctx.eval_slices(p128, bits, ids)[:, 0]
ref = tn.slice_values(tn.ket_network(ops, bits), p128.sliced_wires(), ids[:3], restarts=4, cap_elems=2 ** 25)
print("c128 vs O3 (3 slices)", np.max(np.abs(g128[:3] - ref)) / np.max(np.abs(ref)))
if p64.sliced_wires() == p128.sliced_wires():
    e = np.abs(g64 - g128) / np.abs(g128)
    print("c64 vs c128 per slice rel: max", e.max(), "median", np.median(e), "max-norm", np.max(np.abs(g64 - g128)) / np.max(np.abs(g128)))
a64 = ctx.amplitude(p64, bits); a128 = ctx.amplitude(p128, bits)
print("amp c64 vs c128", abs(a64 - a128) / abs(a128), a128, "sum slices", g128.sum())
