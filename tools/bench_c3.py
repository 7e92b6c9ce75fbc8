"""Config 3 (BASELINE.json configs[2]): Sycamore-53 m=14, a batch of 2^6 amplitudes (open
qubits 0-5 = grid rows 0-1), complex64, sliced across N GPUs.

    python tools/bench_c3.py probe  [--budget-log2 31] [--slices 3]       # 1 GPU: s/slice, memory
    torchrun --nproc-per-node N ... tools/bench_c3.py full --gpus N       # the whole batch

`full` runs ONE tnqvm_amplitudes call over every slice (the product path: rank r owns the
fixed slice groups g = r mod N, per-group complex128 sums, one NCCL allreduce), after a
one-slice warm-up of the same program.  Time = CUDA events on the ctx stream around the
call, max over ranks.  The same plan at every N (every rank plans; SHA-256 compared).
Prints one JSON line (rank 0) and saves the 64 amplitudes to gpurun_out/c3_amps_N<N>.npy
(bit-identity across N is checked on the host afterwards).  Porter-Thomas statistics of
x = 2^53 |a|^2 over the 64 amplitudes are reported (mean ~ 1, mean x^2 ~ 2).
"""
import argparse
import hashlib
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
if os.environ.get("NCCL_DEBUG", "VERSION").upper() == "VERSION":
    os.environ["NCCL_DEBUG"] = "WARN"
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2104_10523_b200 import tnqvm as T  # noqa: E402
from synth import circuits as C  # noqa: E402
from tools.gpu_clocks import GpuClocks  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("mode", choices=["probe", "full"])
ap.add_argument("--gpus", type=int, default=1)
ap.add_argument("--budget-log2", type=int, default=31, help="max intermediate, log2 complex64 elements")
ap.add_argument("--restarts", type=int, default=4096)
ap.add_argument("--slices", type=int, default=3, help="probe: slices to time")
ap.add_argument("--seed", type=int, default=2,
                help="planner seed (2 at 4096 restarts: the fastest measured C3 plan, profiles/r02z_c3_seed_sweep*.jsonl)")
args = ap.parse_args()

world = int(os.environ.get("WORLD_SIZE", "1"))
rank = int(os.environ.get("RANK", "0"))
local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
if world > 1:
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))

ops = C.sycamore53(14, 0)
circ = T.Circuit.from_oplist(ops)
t0 = time.perf_counter()
plan = T.Plan(circ, list(range(6)), 8 << args.budget_log2, seed=args.seed, restarts=args.restarts, dtype=T.C64)
plan_s = time.perf_counter() - t0
info = plan.info()
h = hashlib.sha256(plan.json().encode()).hexdigest()
nccl_id = None
if world > 1:
    hs = [None] * world
    dist.all_gather_object(hs, h)
    assert len(set(hs)) == 1, "plans differ across ranks"
    obj = [T.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    nccl_id = obj[0]
stream = torch.cuda.current_stream()
ctx = T.Context(local, rank, world, nccl_id=nccl_id, stream=stream.cuda_stream)
bits = list(C.random_bitstring(53, 3000))
for q in range(6):
    bits[q] = -1
out = {"config": "c3_sycamore53_m14_open6_c64", "n_gpus": world, "plan_sha256": h[:16], "plan_s": round(plan_s, 1),
       "n_slices": info["n_slices"], "log2_macs_unsliced": round(info["log2_macs_unsliced"], 3),
       "log2_macs_sliced": round(info["log2_macs_sliced"], 3), "flops_sliced": info["flops_sliced"],
       "log2_max_intermediate": info["log2_max_intermediate"], "budget_log2_elems": args.budget_log2,
       "restarts": args.restarts, "planner_seed": args.seed}

if args.mode == "probe":
    ids = list(range(args.slices))
    ctx.eval_slices(plan, bits, ids[:1])  # program build, arena, first-touch
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    vals = ctx.eval_slices(plan, bits, ids)
    e1.record(stream)
    torch.cuda.synchronize()
    dt = e0.elapsed_time(e1) / 1e3 / len(ids)
    out.update({"s_per_slice": dt, "projected_s_1gpu": dt * info["n_slices"],
                "projected_tflops": info["flops_sliced"] / (dt * info["n_slices"]) / 1e12,
                "mem_reserved_GiB": round(torch.cuda.max_memory_reserved() / 2 ** 30, 1),
                "slice_norms": [float(np.linalg.norm(v)) for v in vals]})
    print(json.dumps(out), flush=True)
    sys.exit(0)

# warm-up: one slice of the same program (builds it, sizes the arena and lanes)
ctx.eval_slices(plan, bits, [0])
torch.cuda.synchronize()
if world > 1:
    dist.barrier()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
w0 = time.perf_counter()
with GpuClocks(local) as ck:
    e0.record(stream)
    amps = ctx.amplitudes(plan, bits)
    e1.record(stream)
    torch.cuda.synchronize()
wall = time.perf_counter() - w0
dev_s = e0.elapsed_time(e1) / 1e3
if world > 1:
    t = torch.tensor([dev_s, wall], device="cuda", dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dev_s, wall = float(t[0]), float(t[1])
x = (2.0 ** 53) * np.abs(amps) ** 2
out.update({"seconds": dev_s, "wall_s": wall, "amplitudes_per_s": 64 / dev_s,
            "tflops": info["flops_sliced"] / dev_s / 1e12,
            "porter_thomas": {"mean_x": float(x.mean()), "mean_x2": float((x ** 2).mean()),
                              "window_3sigma": "mean_x 1 +- 0.375, mean_x2 2 +- 1.7"},
            "clocks": ck.summary(),
            "sum_abs2": float((np.abs(amps) ** 2).sum()), "mem_reserved_GiB": round(
                torch.cuda.max_memory_reserved() / 2 ** 30, 1)})
if rank == 0:
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    np.save(os.path.join(ROOT, "gpurun_out", f"c3_amps_N{world}.npy"), amps)
    print(json.dumps(out), flush=True)
ctx.close()
if world > 1:
    dist.destroy_process_group()
