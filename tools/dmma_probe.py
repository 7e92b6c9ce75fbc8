"""complex128 GEMM: DMMA (method 2) vs SIMT DFMA tiled (method 1): time and error."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2104_10523_b200 import tnqvm as T
ctx = T.Context(0)
for (N, K, M) in [(2 ** 16, 256, 256), (4096, 4096, 2048), (2 ** 20, 64, 64), (2 ** 14, 1024, 1024), (128, 2 ** 16, 128)]:
    X = torch.randn((N, K), dtype=torch.complex128, device="cuda")
    Y = torch.randn((K, M), dtype=torch.complex128, device="cuda")
    C = torch.empty((N, M), dtype=torch.complex128, device="cuda")
    ref = X[:2048] @ Y
    for method in (2, 1):
        ctx.gemm(T.C128, method, X.data_ptr(), Y.data_ptr(), C.data_ptr(), N, K, M)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            ctx.gemm(T.C128, method, X.data_ptr(), Y.data_ptr(), C.data_ptr(), N, K, M)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 3
        err = float((C[:2048] - ref).abs().max() / ref.abs().max())
        print(f"c128 N={N} K={K} M={M} method={method} {ms:.3f} ms {8.0*N*K*M/ms/1e9:.2f} TF/s err={err:.2e}", flush=True)
