"""Benchmark: Sycamore-53 random-circuit amplitudes (BASELINE.json configs[1]) through
libtnqvm on 1..8 B200 GPUs (slice-parallel, one NCCL allreduce per amplitude).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    (N>1: python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 ... bench.py --gpus N)

A step = one tnqvm_amplitude_batch call over BENCH_BATCH (8) bitstrings, each a whole
single-amplitude contraction: leaf upload, every pairwise contraction of every slice this
rank owns (each step of the plan ONE launch over slices x bitstrings), complex128 group
accumulation, NCCL allreduce, result copy.  `value` = amplitudes / the summed device span of
the calls (CUDA events on the ctx stream inside the call, leaf upload to result copy);
`e2e` = the same calls timed by CUDA events around them (host network build, pinned
staging, H2D and D2H included); `e2e.single_call_value` = one tnqvm_amplitude call per
bitstring.  The same plan and slicing (min_slices = 8) is used at every GPU count (strong
scaling).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
# NCCL (whatever NCCL_DEBUG the caller sets -- INFO shows the communicator lines) and other
# native libraries may write to fd 1, while the driver reads exactly one JSON line from rank
# 0's stdout: everything but the result line goes to stderr; emit() writes the one JSON line
# to the saved stdout
_STDOUT_FD = os.dup(1)
os.dup2(2, 1)


def emit(line):
    sys.stdout.flush()
    os.write(_STDOUT_FD, (json.dumps(line) + "\n").encode())

METRIC = "Sycamore-53 amplitudes/s & contraction TFLOP/s (% peak) at 1/2/4/8 B200"
UNIT = "amplitudes/s"
CYCLES, CIRCUIT_SEED = 10, 0
# planner seed and restarts: chosen by measuring the winners of 104 (seed, restarts) candidates on B200
# (profiles/r02z_seed_sweep*.jsonl: 129-395 amplitudes/s; the time model ranks them poorly)
PLAN_SEED = int(os.environ.get("BENCH_PLAN_SEED", "2"))  # recorded in the line's config
RESTARTS = int(os.environ.get("BENCH_RESTARTS", "4096"))  # planner restarts (recorded in the config)
BUDGET_BYTES = 16 << 30       # largest intermediate <= 2^31 complex64 elements
MIN_SLICES = int(os.environ.get("BENCH_MIN_SLICES", "8"))


def peaks():
    """(HBM GB/s, bf16 TF/s, source) from the driver's MEASURED_PEAKS.json, else the fallback."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), float(d["bf16_tflops"]), "measured"
    except Exception:  # noqa: BLE001
        return 6650.0, 1590.0, "fallback"


def tensor_peaks():
    """Measured TF32 and FP64 dense peaks of this pool's B200s (tools/measure_peaks.py, cuBLAS
    fp32-with-TF32 and fp64 8192^3 matmuls, burst = best single call at 1965 MHz, no throttle;
    profiles/r02_peaks.json).  The complex64 3xTF32 path's useful peak = TF32 / 3."""
    with open(os.path.join(ROOT, "profiles", "r02_peaks.json")) as f:
        d = json.load(f)
    return float(d["tf32"]["burst_tflops"]), float(d["fp64"]["burst_tflops"]), "profiles/r02_peaks.json (burst)"


class Clocks:
    """SM clock / throttle-reason sampling during the timed region (B200_PROFILING.md clocks
    line): nvidia-smi in a subprocess every 0.2 s.  In-process NVML polling was measured to
    slow this process's kernel launches by ~35%, so it is not used."""

    NAMES = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown", 0x4: "sw_power_cap"}

    def __init__(self, index):
        self.index = index
        self.samples = []  # (sm_mhz, max_mhz, reasons_mask, util)
        self._stop = threading.Event()
        self._t = None

    def _smi(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap,utilization.gpu")
        bits = [0x8, 0x40, 0x20, 0x4]

        def sample():
            out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                  "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                 timeout=5).stdout.strip()
            v = [x.strip() for x in out.split(",")]
            mask = sum(b for b, x in zip(bits, v[2:6]) if x.lower() == "active")
            util = float(v[6]) if v[6] not in ("[N/A]", "") else 0.0
            return float(v[0]), float(v[1]), mask, util
        return sample

    def start(self):
        if os.environ.get("BENCH_NO_CLOCKS"):  # diagnosis only: the JSON line then says "unsampled"
            return
        sample, dt = self._smi(), 0.2

        def run():
            while not self._stop.is_set():
                try:
                    self.samples.append(sample())
                except Exception:  # noqa: BLE001
                    pass
                self._stop.wait(dt)
        self._t = threading.Thread(target=run, daemon=True)
        self._t.start()

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        loaded = sorted(s[0] for s in self.samples if s[3] > 0) or sorted(s[0] for s in self.samples)
        reasons = sorted({n for s in self.samples for b, n in self.NAMES.items() if s[2] & b})
        return {"sm_mhz": loaded[len(loaded) // 2], "sm_max_mhz": float(self.samples[0][1]), "reasons": reasons,
                "samples": len(self.samples)}


def dist_setup(n):
    import torch
    import torch.distributed as dist
    if n <= 1 and int(os.environ.get("WORLD_SIZE", "1")) <= 1:
        return 0, 1, 0
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(n)))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return rank, world, local


def ncu_traffic(cls):
    """DRAM bytes per launch of kernel class `cls` from the newest committed ncu capture
    (profiles/*_traffic.json, written by tools/traffic_summary.py), or None."""
    import glob
    best = None
    for f in sorted(glob.glob(os.path.join(ROOT, "profiles", "r02*_traffic.json"))):
        try:
            d = json.load(open(f))
        except Exception:  # noqa: BLE001
            continue
        if d.get("class") == cls:
            best = (f, d)
    if best is None:
        return None
    return {"bytes_per_launch": best[1]["dram_bytes_per_launch"], "file": os.path.relpath(best[0], ROOT)}


def make_plan(T, C):
    ops = C.sycamore53(CYCLES, CIRCUIT_SEED)
    circ = T.Circuit.from_oplist(ops)
    t0 = time.perf_counter()
    cost_model = int(os.environ.get("BENCH_COST_MODEL", "1"))  # 1 = B200 time model (default), 0 = MACs
    plan = T.Plan(circ, [], BUDGET_BYTES, seed=PLAN_SEED, restarts=RESTARTS, dtype=T.C64, min_slices=MIN_SLICES,
                  cost_model=cost_model)
    return ops, circ, plan, time.perf_counter() - t0


def _oracle_c2_setup(bits):
    """The CPU oracle (O3, numpy complex128) on this workload, set up WITHOUT libtnqvm: the
    plan's sliced wire names are read as data (tests/golden/c2_sliced_wires.json, written by
    tools/plan_data.py c2); O3 builds its own network, fixes those wires per slice and
    contracts along its own greedy order with its own memory sub-slicing."""
    from oracle import einsum_net as tn
    from synth import circuits as C
    with open(os.path.join(ROOT, "tests", "golden", "c2_sliced_wires.json")) as f:
        d = json.load(f)
    ops = C.sycamore53(d["cycles"], d["seed"])
    net = tn.ket_network(ops, bits)
    t0 = time.perf_counter()
    fixed0 = tn.slice_assignment(d["sliced"], 0)
    _, path, sub = tn.subslice_plan(net, fixed0, restarts=8, cap_elems=2 ** 26)
    setup_s = time.perf_counter() - t0
    return tn, net, d, path, sub, setup_s


def _oracle_threads():
    try:
        import threadpoolctl
        return max(p.get("num_threads", 1) for p in threadpoolctl.threadpool_info()) or os.cpu_count()
    except Exception:  # noqa: BLE001
        return os.cpu_count()


def _oracle_steps(setup, nsteps):
    """nsteps oracle steps; step i contracts memory sub-slice (i mod nsub) of GPU slice
    (i div nsub) mod n_slices -- consecutive steps complete whole slices.  Returns the
    per-step seconds and the number of whole slices completed."""
    tn, net, d, path, sub, _ = setup
    nsub = 2 ** len(sub)
    times, cache = [], {}
    for i in range(nsteps):
        s = (i // nsub) % d["n_slices"]
        if s not in cache:
            cache.clear()
            cache[s] = tn._fix(net.tensors, tn.slice_assignment(d["sliced"], s))
        t0 = time.perf_counter()
        tn.contract_subslice(cache[s], path, sub, i % nsub)
        times.append(time.perf_counter() - t0)
    return times, nsteps // nsub


def cpu_baseline(bits, budget_s=20.0):
    """The oracle as it stands on this box's host cores, on a bounded sample of the same
    workload: whole memory sub-slices of the GPU slices for ~budget_s."""
    setup = _oracle_c2_setup(bits)
    tn, net, d, path, sub, setup_s = setup
    nsub = 2 ** len(sub)
    times, cache = [], {}
    t_end = time.perf_counter() + budget_s
    while time.perf_counter() < t_end:
        i = len(times)
        s = (i // nsub) % d["n_slices"]
        if s not in cache:
            cache = {s: tn._fix(net.tensors, tn.slice_assignment(d["sliced"], s))}
        t0 = time.perf_counter()
        tn.contract_subslice(cache[s], path, sub, i % nsub)
        times.append(time.perf_counter() - t0)
    done = len(times)
    per_amp = sum(times) / len(times) * nsub * d["n_slices"]
    return {"value": 1.0 / per_amp, "unit": UNIT, "cores": int(_oracle_threads()), "kind": "oracle",
            "sample": f"O3 numpy complex128 (no libtnqvm): {done} whole memory sub-slices (each 1/{nsub * d['n_slices']} "
                      f"of the amplitude: {nsub} per GPU slice x {d['n_slices']} slices) in {sum(times):.1f}s "
                      f"(+{setup_s:.1f}s own path search)", "seconds_per_amplitude": per_amp,
            "host_cpu_count": os.cpu_count()}


def run_reference(args):
    """--impl reference: the CPU oracle as it stands, timed on this box's host cores (rank 0
    only; other ranks exit).  A step = one whole memory sub-slice of one GPU slice of the
    amplitude (1/32 of it for this plan); consecutive steps complete whole slices."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    bits = [0] * 53
    setup = _oracle_c2_setup(bits)
    tn, net, d, path, sub, setup_s = setup
    nsub = 2 ** len(sub)
    _oracle_steps(setup, args.warmup)
    times, whole = _oracle_steps(setup, args.steps)
    t = sum(times) / len(times)
    per_amp = t * nsub * d["n_slices"]
    line = {"impl": "reference", "metric": METRIC, "value": 1.0 / per_amp, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * t, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "c128", "data": "synthetic",
            "config": {"workload": "sycamore53_m10_single_amplitude", "qubits": 53, "cycles": d["cycles"],
                       "circuit_seed": d["seed"], "bitstring": "0^53", "parallelism": "host cores",
                       "step": f"one O3 memory sub-slice = 1/{nsub * d['n_slices']} amplitude"},
            "cpu_baseline": {"kind": "oracle", "cores": int(_oracle_threads()), "value": 1.0 / per_amp, "unit": UNIT,
                             "sample": f"{args.steps} timed sub-slices ({whole} whole GPU slices), O3 numpy complex128, "
                                       f"own path search {setup_s:.1f}s outside the timing; no libtnqvm in this process"},
            "e2e": {"value": 1.0 / per_amp, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    emit(line)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    from paper_2104_10523_b200 import tnqvm as T
    from synth import circuits as C

    rank, world, local = dist_setup(args.gpus)
    torch.cuda.set_device(local)
    ops, circ, plan, plan_s = make_plan(T, C)
    info = plan.info()
    # every rank plans independently; the plan must be byte-identical everywhere
    import hashlib
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
    # a step = one tnqvm_amplitude_batch call over BATCH single-amplitude bitstrings (C2 is the
    # single-amplitude workload: every bitstring is its own contraction; the batch call runs
    # them through the same launches, slices x bitstrings as the batch dimension)
    BATCH = max(1, int(os.environ.get("BENCH_BATCH", "8")))
    pool = [[0] * 53] + [list(C.random_bitstring(53, 1000 + i)) for i in range(63)]

    def rows(i):
        return [pool[(i * BATCH + j) % len(pool)] for j in range(BATCH)]

    for i in range(args.warmup):
        ctx.amplitude_batch(plan, rows(i))
    for i in range(2):
        ctx.amplitude(plan, pool[i])
    torch.cuda.synchronize()
    clocks = Clocks(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    dev_ms = 0.0
    launches = 0
    h2d = d2h = 0
    e0.record(stream)
    for i in range(args.steps):
        ctx.amplitude_batch(plan, rows(i))
        st = ctx.stats()
        if os.environ.get("BENCH_DEBUG"):
            print(f"step {i} ms_total {st['ms_total']:.3f} host {st['host_ms']:.3f} graph {st['graph']}", file=sys.stderr)
        dev_ms += st["ms_total"]
        launches += st["kernel_launches"]
        h2d += st["h2d_bytes"]
        d2h += st["d2h_bytes"]
    e1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1)
    # single-amplitude calls (tnqvm_amplitude, one bitstring per call), for reference
    e0.record(stream)
    single_dev = 0.0
    for i in range(args.steps):
        ctx.amplitude(plan, pool[i % len(pool)])
        single_dev += ctx.stats()["ms_total"]
    e1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ck = clocks.stop()
    single_ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([e2e_ms, dev_ms, single_ms, single_dev], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms, dev_ms, single_ms, single_dev = float(t[0]), float(t[1]), float(t[2]), float(t[3])
    # instrumented pass right after the timed region (same process, warm): one step's calls
    # with CUDA events around every op on its launch stream (the same launches on the same
    # stream as the timed step, without the graph), summed per kernel class; the dominant
    # class gives the roofline line
    hbm, bf16, src = peaks()
    tf32, fp64, tsrc = tensor_peaks()
    c64_tf = tf32 / 3.0   # useful complex64 flops of the 3xTF32 path: three TF32 MMAs per product
    c128_tf = fp64
    ctx.set_roofline(hbm, c64_tf, c128_tf)
    ctx.set_timing(True)
    ctx.amplitude_batch(plan, rows(0))
    st = ctx.stats()
    cls = ctx.class_stats()
    ctx.set_timing(False)
    tot_cls = sum(c["ms"] for c in cls.values()) or 1.0
    dom = max(cls, key=lambda k: cls[k]["ms"])
    d = cls[dom]
    achieved = d["bytes"] / (d["ms"] * 1e-3) / 1e9 if d["ms"] > 0 else None
    tr = ncu_traffic(dom)
    breakdown = {k: {"ms": round(v["ms"], 4), "share": round(v["ms"] / tot_cls, 4), "ops": v["launches"],
                     "GB_s": round(v["bytes"] / (v["ms"] * 1e-3) / 1e9, 1) if v["ms"] > 0 else None,
                     "TF_s": round(v["flops"] / (v["ms"] * 1e-3) / 1e12, 2) if v["ms"] > 0 else None,
                     "roofline_frac": round(v["roof_ms"] / v["ms"], 4) if v["ms"] > 0 else None}
                 for k, v in cls.items() if v["launches"]}
    roof_tot = sum(v["roof_ms"] for v in cls.values())
    roof_hbm_tot = sum(v["roof_hbm_ms"] for v in cls.values())
    amp_per_s = args.steps * BATCH / (dev_ms * 1e-3)
    flops = info["flops_sliced"]
    line = {
        "metric": METRIC, "value": amp_per_s, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dev_ms / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "c64", "data": "synthetic",
        "config": {"workload": "sycamore53_m10_single_amplitude", "qubits": 53, "cycles": CYCLES,
                   "circuit_seed": CIRCUIT_SEED, "planner_seed": PLAN_SEED, "restarts": RESTARTS,
                   "cost_model": json.loads(plan.json())["cost_model"],
                   "n_slices": info["n_slices"], "log2_macs": round(info["log2_macs_sliced"], 3),
                   "log2_max_intermediate": info["log2_max_intermediate"], "plan_seconds": round(plan_s, 2),
                   "bitstrings_per_step": BATCH,
                   "step": f"one tnqvm_amplitude_batch call over {BATCH} bitstrings (each a whole single-amplitude "
                           "contraction); value = amplitudes / summed device span of the calls (CUDA events on the "
                           "ctx stream, leaf upload to result copy)",
                   "parallelism": f"slices{world}", "l2": "inputs > L2 (intermediates up to 2^"
                   f"{int(info['log2_max_intermediate'])} c64 per slice, 8 slices x {BATCH} bitstrings per launch)"},
        "tflops": flops * BATCH / (dev_ms / args.steps * 1e-3) / 1e12,
        "e2e": {"value": args.steps * BATCH / (e2e_ms * 1e-3), "unit": UNIT, "h2d_bytes_per_step": h2d // args.steps,
                "d2h_bytes_per_step": d2h // args.steps,
                "api": f"tnqvm_amplitude_batch, {BATCH} host bitstrings per call, CUDA events around the calls",
                "single_call_value": args.steps / (single_ms * 1e-3),
                "single_call_device_value": args.steps / (single_dev * 1e-3)},
        "gpu_launches": launches,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                     "frac": (achieved / hbm) if achieved else None,
                     "traffic": tr["bytes_per_launch"] if tr else None,
                     "algorithmic_bytes_per_launch": d["bytes"] / d["launches"] if d["launches"] else None,
                     "traffic_source": (tr["file"] + " (ncu dram__bytes_read.sum + dram__bytes_write.sum per launch, "
                                        "cold cache)") if tr else None,
                     "kernel": dom, "peak_source": src, "share_of_step": d["ms"] / tot_cls,
                     "algorithmic_bytes_per_step": d["bytes"], "launches_per_step": d["launches"],
                     "timing": "instrumented step after the timed region: the same launches on the same stream "
                               "(one launch per step over all slices), CUDA events around each op, no graph",
                     "breakdown": breakdown},
        # SURVEY 8(d) "roofline fraction": sum over ops of max(bytes/HBM, flops/peak) / measured
        "step_roofline": {"frac_instrumented": roof_tot / tot_cls if tot_cls else None,
                          "frac_timed": roof_tot / (dev_ms / args.steps) if dev_ms else None,
                          "roofline_ms": roof_tot, "hbm_bound_share": roof_hbm_tot / roof_tot if roof_tot else None,
                          "peaks": {"hbm_GB_s": hbm, "c64_3xtf32_TF_s": round(c64_tf, 1), "c128_fp64_TF_s": c128_tf,
                                    "source": src + " HBM; " + tsrc + " TF32 / 3 and FP64"}},
        "clocks": ck,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(pool[0])
    if rank == 0:
        emit(line)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
