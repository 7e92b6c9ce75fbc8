import sys, torch
sys.path.insert(0, '.')
from paper_2104_10523_b200 import tnqvm as T
ctx = T.Context(0)
for dtype, td in ((T.C64, torch.complex64), (T.C128, torch.complex128)):
    for (N, K, M) in [(64,16,4),(65,16,4),(75840,16,4),(75904,16,4),(100000,16,4),(2**20,16,4),(2**20,16,8),(2**20,4,4),(2**18,16,16),(2**20,2,2)]:
        X = torch.randn((N, K), dtype=td, device="cuda"); Y = torch.randn((K, M), dtype=td, device="cuda")
        Cm = torch.full((N, M), float('nan'), dtype=td, device="cuda")
        ctx.gemm(dtype, 1, X.data_ptr(), Y.data_ptr(), Cm.data_ptr(), N, K, M)
        ref = X.to(torch.complex128) @ Y.to(torch.complex128)
        d = (Cm.to(torch.complex128) - ref).abs()
        bad = torch.nonzero(torch.isnan(d) | (d > 1e-3 * ref.abs().max()))
        print(dtype, N, K, M, float(torch.nan_to_num(d, 1e9).max()), bad.shape[0], bad[:3].tolist() if bad.shape[0] else "")
