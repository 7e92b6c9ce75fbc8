"""N2 accuracy/time probe: tcgen05 3xTF32 complex64 GEMM vs complex128 torch, error ratio to
torch complex64 (allow_tf32=False), on the N2 test shapes and the C2 step shapes."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2104_10523_b200 import tnqvm as T
torch.backends.cuda.matmul.allow_tf32 = False
ctx = T.Context(0)
shapes = [(128, 2, 8), (1000, 16, 4), (4096, 16, 16), (70001, 64, 32), (33, 256, 64), (5000, 2, 256), (2 ** 20, 16, 8),
          (300, 2048, 128), (128, 4096, 64), (2048, 512, 512), (2 ** 18, 128, 128), (1000, 256, 256), (4224, 128, 32),
          (700, 1024, 16), (2 ** 17, 32, 512), (2 ** 20, 128, 128), (2 ** 20, 128, 64), (2 ** 21, 32, 64), (2 ** 21, 32, 32), (2 ** 19, 64, 64), (2 ** 20, 32, 64), (2 ** 14, 32, 2 ** 11)]
for N, K, M in shapes:
    g = torch.Generator(device="cuda").manual_seed(N * 7 + K * 3 + M)
    X = torch.randn((N, K), dtype=torch.complex64, device="cuda", generator=g)
    Y = torch.randn((K, M), dtype=torch.complex64, device="cuda", generator=g)
    Cm = torch.empty((N, M), dtype=torch.complex64, device="cuda")
    f = lambda: ctx.gemm(T.C64, 2, X.data_ptr(), Y.data_ptr(), Cm.data_ptr(), N, K, M)
    f(); torch.cuda.synchronize()
    ref = X.to(torch.complex128) @ Y.to(torch.complex128)
    sc = ref.abs().max()
    err = float((Cm.to(torch.complex128) - ref).abs().max() / sc)
    e32 = float(((X @ Y).to(torch.complex128) - ref).abs().max() / sc)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20
    e0.record()
    for _ in range(reps): f()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(json.dumps({"tag": os.environ.get("TAG", ""), "N": N, "K": K, "M": M,
                      "err": err, "err32": e32, "ratio": err / e32, "us": ms * 1e3,
                      "TF_s": 8.0 * N * K * M / (ms * 1e-3) / 1e12,
                      "GB_s": 8.0 * (N * K + K * M + N * M) / (ms * 1e-3) / 1e9}), flush=True)
