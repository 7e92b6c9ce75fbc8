"""Per-launch GPU time of the complex GEMM kernels without host launch overhead: R launches
of one shape captured in a CUDA graph on the ctx stream, replayed, timed with CUDA events.

    python tools/tc_graph_probe.py N,K,M [N,K,M ...]       (method 2 = tcgen05 3xTF32)
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2104_10523_b200 import tnqvm as T  # noqa: E402

R = int(os.environ.get("PROBE_REPS", "20"))
method = int(os.environ.get("PROBE_METHOD", "2"))
s = torch.cuda.Stream()
ctx = T.Context(0, stream=s.cuda_stream)
for arg in sys.argv[1:]:
    N, K, M = (int(v) for v in arg.split(","))
    X = torch.randn((N, K), dtype=torch.complex64, device="cuda")
    Y = torch.randn((K, M), dtype=torch.complex64, device="cuda")
    C = torch.empty((N, M), dtype=torch.complex64, device="cuda")
    with torch.cuda.stream(s):
        for _ in range(3):
            ctx.gemm(T.C64, method, X.data_ptr(), Y.data_ptr(), C.data_ptr(), N, K, M)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(R):
            ctx.gemm(T.C64, method, X.data_ptr(), Y.data_ptr(), C.data_ptr(), N, K, M)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(5):
        g.replay()
    e1.record(s)
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / (5 * R)
    flops = 8.0 * N * K * M
    byts = 8.0 * (N * K + K * M + N * M)
    print(f"N={N} K={K} M={M} method={method} {us:.2f} us/launch {flops / us / 1e6:.1f} TF/s "
          f"{byts / us / 1e3:.1f} GB/s pdl={os.environ.get('TNQVM_PDL', '1')}", flush=True)
