"""N1 permute kernel sweep: rank-r binary tensors under seeded random permutations and
'skinny GEMM operand' permutations; GB/s = 2*bytes/time vs the measured HBM copy peak."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2104_10523_b200 import tnqvm as T

ctx = T.Context(0)
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"]
res = []
for dtype, td in ((T.C64, torch.complex64), (T.C128, torch.complex128)):
    for rank in (24, 28, 30):
        if dtype == T.C128 and rank > 29:
            continue
        x = torch.randn((2,) * rank, dtype=td, device="cuda")
        y = torch.empty_like(x)
        rng = np.random.default_rng(rank)
        perms = [("random%d" % i, rng.permutation(rank)) for i in range(4)]
        # skinny operand: move 3..8 scattered modes to the end (contracted modes fastest)
        for k in (3, 6):
            sel = sorted(rng.choice(rank, k, replace=False))
            perms.append((f"tofront{k}", np.array([m for m in range(rank) if m not in sel] + list(sel))))
        for name, perm in perms:
            ctx.permute(dtype, x.data_ptr(), y.data_ptr(), rank, perm)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(5):
                ctx.permute(dtype, x.data_ptr(), y.data_ptr(), rank, perm)
            e1.record(); torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 5
            gbs = 2 * x.numel() * x.element_size() / ms / 1e6
            ok = bool(torch.equal(y, x.permute(*[int(p) for p in perm]).contiguous())) if rank <= 24 else None
            res.append({"dtype": "c64" if dtype == T.C64 else "c128", "rank": rank, "perm": name, "ms": ms, "GBps": gbs, "frac": gbs / peak, "exact": ok})
            print(json.dumps(res[-1]), flush=True)
        del x, y
        torch.cuda.empty_cache()
v = sorted(r["GBps"] for r in res)
print(json.dumps({"median_GBps": v[len(v) // 2], "peak": peak, "median_frac": v[len(v) // 2] / peak}))
