"""One canonical (K-contiguous, TMA) tcgen05 GEMM and one gather GEMM of the same shape, for
an ncu side-by-side (diagnostics).  usage: python tools/gemm_pair_probe.py "<layout>" nm"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2104_10523_b200 import tnqvm as T  # noqa: E402

order = sys.argv[1].split()
nm = int(sys.argv[2])
nn = sum(b[0] == "n" for b in order)
nk = sum(b[0] == "k" for b in order)
N, K, M = 2 ** nn, 2 ** nk, 2 ** nm
pos = {b: i for i, b in enumerate(order)}
ctx = T.Context(0)
X = torch.randn(N * K, dtype=torch.complex64, device="cuda")
Y = torch.randn((K, M), dtype=torch.complex64, device="cuda")
Cm = torch.empty((N, M), dtype=torch.complex64, device="cuda")
ctx.gemm(T.C64, 2, X.data_ptr(), Y.data_ptr(), Cm.data_ptr(), N, K, M)
ctx.gemm_gather(T.C64, X.data_ptr(), Y.data_ptr(), Cm.data_ptr(), nn, nk, nm,
                [2 ** pos[f"n{i}"] for i in range(nn)], [2 ** pos[f"k{i}"] for i in range(nk)])
torch.cuda.synchronize()
print("ok")
