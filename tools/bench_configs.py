"""Secondary measurements for the other BASELINE.json configs (not the driver's bench line):
C1 GHZ+QFT 8q, C3 Sycamore-53 m=14 with 2^6 open (slice subset, projected), C4 QAOA 40q p=2,
C5 20-qubit noisy doubled network.  Each is checked against the oracle where affordable.
Prints one JSON line per config."""
import json
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import lightcone as lc  # noqa: E402
from oracle import statevector as sv  # noqa: E402
from paper_2104_10523_b200 import tnqvm as T  # noqa: E402
from synth import circuits as C  # noqa: E402
from tools.gpu_clocks import GpuClocks  # noqa: E402

which = sys.argv[1:] or ["c1", "c4", "c5", "c3"]
CM = int(os.environ.get("COST_MODEL", "1"))  # planner objective for every config below
ctx = T.Context(0)


CLK = {}


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    with GpuClocks(0) as ck:
        t = time.perf_counter()
        for _ in range(reps):
            r = fn()
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t) / reps
    CLK["last"] = ck.summary()
    return dt, r


if "c1" in which:
    ops = C.ghz_qft(8)
    p = T.Plan(T.Circuit.from_oplist(ops), list(range(8)), 1 << 30, dtype=T.C128, restarts=16)
    dt, v = timed(lambda: ctx.amplitudes(p, [-1] * 8), 50)
    st = ctx.stats()
    ref = sv.evolve(ops)
    print(json.dumps({"config": "c1_ghz_qft8_all256_c128", "us_per_call": dt * 1e6, "device_us": st["ms_total"] * 1e3,
                      "amplitudes_per_s": 256 / dt, "kernel_launches": st["kernel_launches"],
                      "max_rel_err_vs_O1": float(np.max(np.abs(v - ref)) / np.max(np.abs(ref))),
                      "clocks": CLK["last"]}), flush=True)

if "c4" in which:
    ops, terms = C.qaoa40(0)
    circ = T.Circuit.from_oplist(ops)
    for dtype, name in ((T.C128, "c128"), (T.C64, "c64")):
        dt, (tot, per) = timed(lambda: ctx.expectation(circ, terms, per_term=True, dtype=dtype, restarts=16), 5)
        st = ctx.stats()
        ref_tot, ref_per = lc.expectation(ops, terms)
        pk = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                                         "r02_peaks.json")))
        simt = pk["fp32_simt"]["burst_tflops"] if dtype == T.C64 else pk["fp64"]["burst_tflops"]
        print(json.dumps({"config": f"c4_qaoa40_p2_{name}", "ms_per_H": dt * 1e3, "device_ms": st["ms_total"],
                          "batch_kernel_tflops": st["flops"] / (st["ms_total"] * 1e-3) / 1e12,
                          "frac_of_simt_peak": st["flops"] / (st["ms_total"] * 1e-3) / 1e12 / simt,
                          "simt_peak_tflops": simt, "simt_peak_source": "profiles/r02_peaks.json " +
                          ("fp32 sgemm without TF32" if dtype == T.C64 else "fp64 (DMMA; upper bound for FP64 FMA)"),
                          "H_evals_per_s": 1 / dt, "terms_per_s": len(terms) / dt, "value": tot.real,
                          "maxcut_value": len(terms) / 2 - tot.real / 2, "kernel_launches": st["kernel_launches"],
                          "max_rel_err_per_term": float(np.max(np.abs(per - np.array(ref_per))) / np.max(np.abs(ref_per))),
                          "clocks": CLK["last"]}),
              flush=True)

if "c5" in which:
    ops = C.noisy_grid_circuit(4, 5, 8, 0)
    circ = T.Circuit.from_oplist(ops)
    t0 = time.perf_counter()
    p = T.Plan(circ, [], 16 << 31, dtype=T.C128, restarts=64, cost_model=CM)
    plan_s = time.perf_counter() - t0
    info = p.info()
    bits = [list(C.random_bitstring(20, 2000 + i)) for i in range(4)]
    probs = []
    ctx.amplitude(p, bits[0])
    torch.cuda.synchronize()
    dev_ms = 0
    with GpuClocks(0) as ck:
        t = time.perf_counter()
        for b in bits:
            probs.append(ctx.amplitude(p, b))
            dev_ms += ctx.stats()["ms_total"]
        dt = (time.perf_counter() - t) / len(bits)
    print(json.dumps({"config": "c5_noisy20_m8_c128", "s_per_probability": dt, "probabilities_per_s": 1 / dt,
                      "tflops": info["flops_sliced"] / (dev_ms / len(bits) * 1e-3) / 1e12,
                      "log2_macs": info["log2_macs_sliced"], "plan_s": plan_s,
                      "probs": [pp.real for pp in probs], "max_imag": max(abs(pp.imag) for pp in probs),
                      "clocks": ck.summary()}), flush=True)

if "c3" in which:
    ops = C.sycamore53(14, 0)
    circ = T.Circuit.from_oplist(ops)
    t0 = time.perf_counter()
    p = T.Plan(circ, list(range(6)), 8 << 32, restarts=int(os.environ.get("C3_RESTARTS", "64")), seed=0, cost_model=CM)
    plan_s = time.perf_counter() - t0
    info = p.info()
    bits = list(C.random_bitstring(53, 3000))
    for q in range(6):
        bits[q] = -1
    ids = list(range(min(8, info["n_slices"])))
    ctx.eval_slices(p, bits, ids[:1])
    torch.cuda.synchronize()
    with GpuClocks(0) as ck:
        t = time.perf_counter()
        vals = ctx.eval_slices(p, bits, ids)
        dt = (time.perf_counter() - t) / len(ids)
    full = dt * info["n_slices"]
    print(json.dumps({"config": "c3_sycamore53_m14_open6_c64", "s_per_slice": dt, "n_slices": info["n_slices"],
                      "projected_s_1gpu": full, "projected_amplitudes_per_s_1gpu": 64 / full,
                      "projected_amplitudes_per_s_8gpu_ideal": 8 * 64 / full,
                      "log2_macs_sliced": info["log2_macs_sliced"], "flops_sliced": info["flops_sliced"],
                      "tflops": info["flops_sliced"] / full / 1e12, "plan_s": plan_s,
                      "slice_norms": [float(np.linalg.norm(v)) for v in vals[:2]], "clocks": ck.summary()}), flush=True)
