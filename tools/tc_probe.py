"""tcgen05 3xTF32 GEMM: accuracy vs fp32 cgemm and timing per shape (CUDA events)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2104_10523_b200 import tnqvm as T  # noqa: E402

torch.backends.cuda.matmul.allow_tf32 = False
ctx = T.Context(0)
shapes = [(2 ** 16, 2 ** 11, 2 ** 12), (2 ** 10, 2 ** 18, 2 ** 8), (2 ** 17, 2 ** 9, 2 ** 10), (2 ** 22, 16, 16),
          (2 ** 24, 8, 8), (2 ** 20, 64, 64), (2 ** 18, 256, 256), (4096, 4096, 4096)]
if len(sys.argv) > 1:
    shapes = [tuple(int(x) for x in s.split(",")) for s in sys.argv[1:]]
for (N, K, M) in shapes:
    X = torch.randn((N, K), dtype=torch.complex64, device="cuda")
    Y = torch.randn((K, M), dtype=torch.complex64, device="cuda")
    C = torch.empty((N, M), dtype=torch.complex64, device="cuda")
    for method in (2, 1):
        ctx.gemm(T.C64, method, X.data_ptr(), Y.data_ptr(), C.data_ptr(), N, K, M)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 3
        e0.record()
        for _ in range(reps):
            ctx.gemm(T.C64, method, X.data_ptr(), Y.data_ptr(), C.data_ptr(), N, K, M)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        flops = 8.0 * N * K * M
        byts = 8.0 * (N * K + K * M + N * M)
        err = None
        if N * M <= 2 ** 26 and N * K <= 2 ** 27:
            ref = X[:4096].to(torch.complex128) @ Y.to(torch.complex128)
            err = float((C[:4096].to(torch.complex128) - ref).abs().max() / ref.abs().max())
            e32 = float(((X[:4096] @ Y).to(torch.complex128) - ref).abs().max() / ref.abs().max())
        print(f"N={N} K={K} M={M} method={method} {ms:.3f} ms {flops / ms / 1e9:.1f} TF/s "
              f"{byts / ms / 1e6:.1f} GB/s err={err} fp32_err={e32 if err is not None else None}"
              f" group={os.environ.get('TNQVM_TC_GROUP', 'default')}", flush=True)
        if method == 2 and K * M > 2 ** 22:
            break
