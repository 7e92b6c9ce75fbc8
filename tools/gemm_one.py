"""One tcgen05 GEMM launch of a given shape (diagnostics, for ncu).  usage: gemm_one.py log2N K M"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2104_10523_b200 import tnqvm as T  # noqa: E402

n, K, M = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
N = 2 ** n
ctx = T.Context(0)
X = torch.randn((N, K), dtype=torch.complex64, device="cuda")
Y = torch.randn((K, M), dtype=torch.complex64, device="cuda")
Cm = torch.empty((N, M), dtype=torch.complex64, device="cuda")
for _ in range(2):
    ctx.gemm(T.C64, 2, X.data_ptr(), Y.data_ptr(), Cm.data_ptr(), N, K, M)
torch.cuda.synchronize()
print("ok")
