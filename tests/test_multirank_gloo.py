"""N>1 host path on CPU (world_size 2, gloo): every rank plans independently and must get a
byte-identical plan; the slice groups owned by the ranks partition the slice range; the
NCCL unique id travels by torch.distributed object broadcast (as in bench.py); the
max-over-ranks timing reduction.  (The device allreduce itself is exercised on GPUs.)"""
import hashlib
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        from paper_2104_10523_b200 import tnqvm as T
        from synth import circuits as C
        c = T.Circuit.from_oplist(C.sycamore53(8, 0))
        p = T.Plan(c, [], 16 << 30, restarts=16, seed=3, min_slices=16, threads=1 + rank)
        h = hashlib.sha256(p.json().encode()).hexdigest()
        hs = [None] * world
        dist.all_gather_object(hs, h)
        mine = p.rank_slices(rank, world)
        allv = [None] * world
        dist.all_gather_object(allv, mine)
        obj = [b"x" * 128 if rank == 0 else None]      # stands in for tnqvm_nccl_unique_id()
        dist.broadcast_object_list(obj, src=0)
        t = torch.tensor([10.0 + rank, 1.0 * rank])
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        q.put((rank, len(set(hs)), sorted(s for v in allv for s in v), p.info()["n_slices"], obj[0], t.tolist()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_two_rank_plan_and_partition(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, distinct, slices, n, idb, t in out:
        assert distinct == 1                      # byte-identical plans on every rank
        assert slices == list(range(n))           # groups partition the slice range
        assert idb == b"x" * 128
        assert t == [10.0 + world - 1, world - 1.0]
