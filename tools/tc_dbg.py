import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2104_10523_b200 import tnqvm as T
ctx = T.Context(0)
for N, K, M in [(2 ** 20, 16, 8), (2 ** 21, 32, 32), (2 ** 21, 32, 64), (2 ** 20, 128, 128)]:
    X = torch.randn((N, K), dtype=torch.complex64, device="cuda")
    Y = torch.randn((K, M), dtype=torch.complex64, device="cuda")
    Cm = torch.empty((N, M), dtype=torch.complex64, device="cuda")
    for _ in range(2):
        ctx.gemm(T.C64, 2, X.data_ptr(), Y.data_ptr(), Cm.data_ptr(), N, K, M)
    torch.cuda.synchronize()
