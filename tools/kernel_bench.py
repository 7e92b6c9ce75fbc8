"""Kernel-level benches of SURVEY 8(d) (N1 permute, N2 tcgen05 complex64 GEMM, N3 DMMA
complex128 GEMM): timing with CUDA events over back-to-back stream-ordered launches, errors
against torch complex128, one JSON line per case plus a markdown table (stdout).

    python tools/kernel_bench.py [n1] [n2] [n3]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2104_10523_b200 import tnqvm as T  # noqa: E402
from tools.gpu_clocks import GpuClocks  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
try:
    PK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    HBM = float(PK["hbm_gbs"])
except Exception:  # noqa: BLE001
    HBM = 6650.0
_TP = json.load(open(os.path.join(ROOT, "profiles", "r02_peaks.json")))  # measured (tools/measure_peaks.py)
TF32 = float(_TP["tf32"]["burst_tflops"])  # cuBLAS TF32, burst, 1965 MHz
C64_USEFUL = TF32 / 3.0                   # 3xTF32: three TF32 MMAs per useful product
FP64 = float(_TP["fp64"]["burst_tflops"])  # cuBLAS FP64 (DMMA)
which = sys.argv[1:] or ["n1", "n2", "n3"]
torch.backends.cuda.matmul.allow_tf32 = False
ctx = T.Context(0)
rows = []


CLK = {}


def timeit(fn, reps):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with GpuClocks(0, dt=0.05) as ck:
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
    CLK["last"] = ck.summary()
    return e0.elapsed_time(e1) / reps


def emit(d):
    d = dict(d)
    d.setdefault("clocks", CLK.get("last"))
    rows.append(d)
    print(json.dumps(d), flush=True)


if "n1" in which:
    res = []
    for dtype, td, ranks in ((T.C64, torch.complex64, (24, 28, 30, 32)), (T.C128, torch.complex128, (24, 28, 30))):
        for rank in ranks:
            x = torch.randn((1 << rank,), dtype=td, device="cuda")
            y = torch.empty_like(x)
            rng = np.random.default_rng(rank)
            perms = [("random%02d" % i, rng.permutation(rank)) for i in range(16)]
            for k in (3, 6, 10):  # skinny GEMM operand: scattered modes moved fastest
                sel = sorted(rng.choice(rank, k, replace=False))
                perms.append((f"move{k}", np.array([m for m in range(rank) if m not in sel] + list(sel))))
            for name, perm in perms:
                ms = timeit(lambda: ctx.permute(dtype, x.data_ptr(), y.data_ptr(), rank, perm), 3)
                nbytes = 2 * x.numel() * x.element_size()
                ok = None
                if rank <= 24:  # torch tensors stop at 25 dims
                    xs = x.view((2,) * rank)
                    ok = bool(torch.equal(y.view((2,) * rank), xs.permute(*[int(p) for p in perm]).contiguous()))
                res.append((nbytes, nbytes / ms / 1e6))
                emit({"kernel": "N1 permute_kernel_v3", "dtype": "c64" if dtype == T.C64 else "c128", "rank": rank,
                      "perm": name, "ms": round(ms, 4), "GB_s": round(nbytes / ms / 1e6, 1),
                      "frac_hbm": round(nbytes / ms / 1e6 / HBM, 3), "bit_exact": ok})
            del x, y
            torch.cuda.empty_cache()
    # size-weighted median GB/s
    res.sort(key=lambda t: t[1])
    tot = sum(b for b, _ in res)
    acc = 0
    for b, g in res:
        acc += b
        if acc >= tot / 2:
            emit({"kernel": "N1 summary", "size_weighted_median_GB_s": round(g, 1), "frac_hbm": round(g / HBM, 3),
                  "cases": len(res)})
            break


def gemm_case(dtype, method, N, K, M, label):
    td = torch.complex64 if dtype == T.C64 else torch.complex128
    g = torch.Generator(device="cuda").manual_seed(N + 3 * K + 7 * M)
    X = torch.randn((N, K), dtype=td, device="cuda", generator=g)
    Y = torch.randn((K, M), dtype=td, device="cuda", generator=g)
    Cm = torch.empty((N, M), dtype=td, device="cuda")
    reps = 3 if N * K * M >= 2 ** 33 else 10
    ms = timeit(lambda: ctx.gemm(dtype, method, X.data_ptr(), Y.data_ptr(), Cm.data_ptr(), N, K, M), reps)
    flops = 8.0 * N * K * M
    nbytes = X.element_size() * (N * K + K * M + N * M)
    ai = flops / nbytes
    sub = min(N, 4096)
    ref = X[:sub].to(torch.complex128) @ Y.to(torch.complex128)
    err = float((Cm[:sub].to(torch.complex128) - ref).norm() / ref.norm())
    d = {"kernel": label, "N": N, "K": K, "M": M, "ms": round(ms, 4), "TF_s": round(flops / ms / 1e9, 1),
         "GB_s": round(nbytes / ms / 1e6, 1), "AI_flop_per_B": round(ai, 1), "frob_rel_err": err}
    if dtype == T.C64:
        e32 = float(((X[:sub] @ Y).to(torch.complex128) - ref).norm() / ref.norm())
        d["err_vs_fp32_matmul"] = round(err / e32, 2)
        ridge = C64_USEFUL * 1e3 / HBM
        d["bound"] = "tensor" if ai >= ridge else "hbm"
        d["frac"] = round(flops / ms / 1e9 / C64_USEFUL, 3) if ai >= ridge else round(nbytes / ms / 1e6 / HBM, 3)
    else:
        ridge = FP64 * 1e3 / HBM
        d["bound"] = "fp64" if ai >= ridge else "hbm"
        d["frac"] = round(flops / ms / 1e9 / FP64, 3) if ai >= ridge else round(nbytes / ms / 1e6 / HBM, 3)
    emit(d)
    del X, Y, Cm
    torch.cuda.empty_cache()


if "n2" in which:
    for n in (11, 12, 13):
        gemm_case(T.C64, 2, 2 ** n, 2 ** n, 2 ** n, "N2 tcgen05 3xTF32 square")
    for m in (3, 4, 5, 6, 7):
        for k in (3, 4, 5, 6, 7, 8):
            gemm_case(T.C64, 2, 2 ** 24, 2 ** k, 2 ** m, "N2 tcgen05 3xTF32 skinny")
if "n2c" in which:  # every tensor-core step shape of the C2 / C3 programs at its real size (trace_c2, bench_c3)
    C2 = [(17, 7, 7), (17, 7, 6), (18, 5, 6), (18, 5, 5), (17, 5, 6), (16, 6, 6), (11, 5, 11), (14, 5, 7), (13, 4, 6)]
    C3 = [(22, 8, 9), (22, 9, 8), (21, 10, 7), (25, 6, 6), (24, 7, 6), (23, 7, 7), (21, 6, 10), (24, 6, 6), (22, 8, 6),
          (23, 5, 8)]
    for tag, shapes in (("C2", C2), ("C3", C3)):
        for n, k, m in shapes:
            gemm_case(T.C64, 2, 2 ** n, 2 ** k, 2 ** m, f"N2 tcgen05 3xTF32 {tag} step")
if "n2b" in which:  # the C2 tensor-core steps as the bench launches them: 16 units per launch (N x 16)
    for n, k, m in [(21, 7, 7), (21, 7, 6), (22, 5, 6), (22, 5, 5), (21, 5, 6), (20, 6, 6), (15, 5, 11), (18, 5, 7),
                    (17, 4, 6)]:
        gemm_case(T.C64, 2, 2 ** n, 2 ** k, 2 ** m, "N2 tcgen05 3xTF32 C2 step x16 units")
def gather_case(order, label):
    """X in the layout `order` (its bits fastest-first, e.g. ['k0', 'n0', ..]): C = X Y through
    the tcgen05 kernel's gather producer; error against torch complex128 on the same X."""
    nn = sum(1 for b in order if b[0] == "n")
    nk = sum(1 for b in order if b[0] == "k")
    N, K, M = 2 ** nn, 2 ** nk, 2 ** order_m[label]
    pos = {b: i for i, b in enumerate(order)}
    sxn = [2 ** pos[f"n{i}"] for i in range(nn)]
    sxk = [2 ** pos[f"k{i}"] for i in range(nk)]
    g = torch.Generator(device="cuda").manual_seed(N + 3 * K + 7 * M)
    Xf = torch.randn(N * K, dtype=torch.complex64, device="cuda", generator=g)
    Y = torch.randn((K, M), dtype=torch.complex64, device="cuda", generator=g)
    Cm = torch.empty((N, M), dtype=torch.complex64, device="cuda")
    ms = timeit(lambda: ctx.gemm_gather(T.C64, Xf.data_ptr(), Y.data_ptr(), Cm.data_ptr(), nn, nk, order_m[label],
                                        sxn, sxk), 5)
    # reference: the flat buffer as a (2,)*r tensor (slowest first), permuted to [n.., k..] row-major
    r = nn + nk
    slow = list(reversed(order))
    perm = [slow.index(f"n{i}") for i in reversed(range(nn))] + [slow.index(f"k{i}") for i in reversed(range(nk))]
    Xm = Xf.view((2,) * r).permute(perm).reshape(N, K)
    sub = min(N, 4096)
    ref = Xm[:sub].to(torch.complex128) @ Y.to(torch.complex128)
    err = float((Cm[:sub].to(torch.complex128) - ref).norm() / ref.norm())
    e32 = float(((Xm[:sub] @ Y).to(torch.complex128) - ref).norm() / ref.norm())
    nbytes = 8 * (N * K + K * M + N * M)
    emit({"kernel": label, "N": N, "K": K, "M": M, "ms": round(ms, 4), "GB_s": round(nbytes / ms / 1e6, 1),
          "frac": round(nbytes / ms / 1e6 / HBM, 3), "bound": "hbm", "frob_rel_err": err,
          "err_vs_fp32_matmul": round(err / e32, 2)})
    del Xf, Y, Cm
    torch.cuda.empty_cache()


# the C2 gather steps' X layouts (bench plan, 16 units merged into the row bits)
def _lay(s):
    return s.split()


order_m = {}
GATHER = {  # generated from the bench plan's program (ops 9, 12-15, 22, 23); 4 unit bits on top
    "C2 op9 gather": (_lay("k0 k1 k2 n0 n1 n2 n3 n4 n5 n6 n7 n8 n9 n10 k3 k4 n11 k5 n12 n13 n14 n15 n16 n17 n18 n19"), 6),
    "C2 op12 gather": (_lay("k0 n0 n1 n2 n3 n4 k1 n5 n6 n7 n8 n9 n10 n11 n12 k2 n13 n14 n15 k3 k4 n16 n17 n18 n19 n20 "
                            "n21"), 5),
    "C2 op13 gather": (_lay("k0 n0 n1 n2 n3 n4 k1 n5 k2 n6 n7 n8 n9 n10 n11 n12 n13 k3 k4 n14 n15 n16 n17 n18 n19 n20 "
                            "n21"), 6),
    "C2 op14 gather": (_lay("k0 n0 n1 n2 n3 n4 n5 n6 n7 n8 n9 k1 n10 k2 n11 n12 n13 n14 n15 n16 k3 k4 k5 k6 n17 n18 n19 "
                            "n20"), 7),
    "C2 op15 gather": (_lay("k0 k1 k2 n0 n1 n2 n3 n4 k3 k4 n5 n6 n7 n8 n9 n10 n11 k5 n12 n13 n14 k6 n15 n16 n17 n18 n19 "
                            "n20"), 6),
    "C2 op22 gather": (_lay("k0 n0 k1 n1 n2 n3 n4 n5 n6 n7 k2 n8 n9 n10 k3 n11 n12 n13 n14 n15 n16"), 6),
    "C2 op23 gather": (_lay("k0 n0 n1 n2 n3 n4 n5 n6 k1 n7 k2 n8 n9 k3 n10 n11 n12 k4 n13 n14 n15 n16 n17"), 7),
    # op13's shape with K-contiguous X, through the gather producer (compare n2b's TMA-producer line)
    "C2 op13 shape, K-contiguous": (_lay("k0 k1 k2 k3 k4 " + " ".join(f"n{i}" for i in range(22))), 6),
}
for _k, (_o, _m) in GATHER.items():
    order_m[_k] = _m
if "n2g" in which:
    for label, (order, _) in GATHER.items():
        gather_case(order, label)
if "n3" in which:
    for n in (11, 12):
        gemm_case(T.C128, 2, 2 ** n, 2 ** n, 2 ** n, "N3 DMMA square")
    for m in (3, 5, 7):
        for k in (3, 5, 8):
            gemm_case(T.C128, 2, 2 ** 22, 2 ** k, 2 ** m, "N3 DMMA skinny")

# markdown summary
print("\n| kernel | shape | ms | GB/s | TF/s | bound | frac | err |")
print("|---|---|---|---|---|---|---|---|")
for d in rows:
    if d["kernel"].startswith("N1 permute"):
        print(f"| {d['kernel']} {d['dtype']} | rank {d['rank']} {d['perm']} | {d['ms']} | {d['GB_s']} | | hbm | "
              f"{d['frac_hbm']} | bit-exact={d['bit_exact']} |")
    elif d["kernel"] == "N1 summary":
        print(f"| N1 size-weighted median | {d['cases']} cases | | {d['size_weighted_median_GB_s']} | | hbm | "
              f"{d['frac_hbm']} | |")
    else:
        print(f"| {d['kernel']} | {d['N']}x{d['K']}x{d['M']} | {d['ms']} | {d['GB_s']} | {d['TF_s']} | {d['bound']} | "
              f"{d['frac']} | {d['frob_rel_err']:.2e}" + (f" ({d['err_vs_fp32_matmul']}x fp32)" if "err_vs_fp32_matmul" in d
                                                          else "") + " |")
