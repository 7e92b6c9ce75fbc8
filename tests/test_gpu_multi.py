"""Multi-GPU slice-parallel path (a10): one process per GPU over NCCL; amplitudes must be
BIT-identical to the 1-GPU result (8 fixed slice groups + one allreduce of zero-padded
group slots); likewise the per-term expectation values.  Skipped unless
>= 2 GPUs are visible."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _expectation(ctx, T, C):
    """QAOA-40 p=2 bra-ket terms (config 4), batched into one small-tensor launch; the
    terms are split over ranks and the per-term values must not depend on the split."""
    ops, terms = C.qaoa40(0)
    tot, per = ctx.expectation(T.Circuit.from_oplist(ops), terms[:12], per_term=True, dtype=T.C64, restarts=8)
    return np.concatenate([[tot], per])


def _worker(rank, world, port, q):
    import sys
    import torch
    import torch.distributed as dist
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2104_10523_b200 import tnqvm as T
    from synth import circuits as C
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    try:
        obj = [T.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        ctx = T.Context(rank, rank, world, nccl_id=obj[0])
        out = []
        for dtype in (T.C64, T.C128):
            c = T.Circuit.from_oplist(C.grid_rqc(4, 5, 10, seed=2))
            p = T.Plan(c, [0, 19], 16 << 12, restarts=8, min_slices=16, dtype=dtype)
            bits = list(C.random_bitstring(20, 1003))
            bits[0] = bits[19] = -1
            out.append(ctx.amplitudes(p, bits))
        out.append(_expectation(ctx, T, C))
        q.put((rank, [o.tobytes() for o in out]))
        ctx.close()
    finally:
        dist.destroy_process_group()


def test_multi_gpu_bit_identical():
    import torch
    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    from paper_2104_10523_b200 import tnqvm as T
    from synth import circuits as C
    ref = []
    ctx = T.Context(0)
    for dtype in (T.C64, T.C128):
        c = T.Circuit.from_oplist(C.grid_rqc(4, 5, 10, seed=2))
        p = T.Plan(c, [0, 19], 16 << 12, restarts=8, min_slices=16, dtype=dtype)
        bits = list(C.random_bitstring(20, 1003))
        bits[0] = bits[19] = -1
        ref.append(ctx.amplitudes(p, bits).tobytes())
    ref.append(_expectation(ctx, T, C).tobytes())
    ctx.close()
    import torch.multiprocessing as mp
    for world in sorted({2, min(n, 4), min(n, 8)}):
        mpc = mp.get_context("spawn")
        q = mpc.Queue()
        port = _free_port()
        procs = [mpc.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
        for pr in procs:
            pr.start()
        res = [q.get(timeout=600) for _ in range(world)]
        for pr in procs:
            pr.join(timeout=120)
            assert pr.exitcode == 0
        for rank, outs in res:
            for a, b in zip(outs, ref):
                assert a == b, f"world {world} rank {rank}: not bit-identical " \
                               f"{np.frombuffer(a, complex)[:2]} vs {np.frombuffer(b, complex)[:2]}"
