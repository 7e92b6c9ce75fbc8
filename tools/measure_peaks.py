"""Measure the tensor-core peaks the roofline needs on THIS box:
TF32 (fp32 matmul with allow_tf32, cuBLAS) and FP64 (float64 matmul, DMMA) dense
throughput, burst (best of 10) and sustained (back to back for ~4 s), with nvidia-smi
clocks and throttle reasons sampled during each run.  Also the HBM copy bandwidth
(b.copy_(a), read + write bytes) for cross-checking MEASURED_PEAKS.json.

    python tools/measure_peaks.py > profiles/r02_peaks.json
"""
import json
import os
import subprocess
import sys
import threading
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


class Clocks:
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,utilization.gpu,power.draw")

    def __init__(self):
        self.s = []
        self.stop_ev = threading.Event()

    def __enter__(self):
        def run():
            while not self.stop_ev.is_set():
                try:
                    out = subprocess.run(["nvidia-smi", "-i", "0", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits"],
                                         capture_output=True, text=True, timeout=5).stdout.strip()
                    self.s.append([x.strip() for x in out.split(",")])
                except Exception:  # noqa: BLE001
                    pass
                self.stop_ev.wait(0.2)
        self.t = threading.Thread(target=run, daemon=True)
        self.t.start()
        return self

    def __exit__(self, *a):
        self.stop_ev.set()
        self.t.join(10)

    def summary(self):
        load = [float(v[0]) for v in self.s if v[6] not in ("", "[N/A]") and float(v[6]) > 0] or [float(v[0]) for v in self.s]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for v in self.s for i in range(4) if v[2 + i].lower() == "active"})
        load.sort()
        return {"sm_mhz_median": load[len(load) // 2] if load else None,
                "sm_max_mhz": float(self.s[0][1]) if self.s else None, "reasons": reasons, "samples": len(self.s),
                "power_w_max": max((float(v[7]) for v in self.s if v[7] not in ("", "[N/A]")), default=None)}


def gemm_rate(dtype, n, tf32):
    torch.backends.cuda.matmul.allow_tf32 = tf32
    a = torch.randn(n, n, device="cuda", dtype=dtype)
    b = torch.randn(n, n, device="cuda", dtype=dtype)
    c = torch.empty(n, n, device="cuda", dtype=dtype)
    flops = 2.0 * n ** 3
    for _ in range(3):
        torch.matmul(a, b, out=c)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 0.0
    with Clocks() as ck_b:
        for _ in range(10):
            e0.record()
            torch.matmul(a, b, out=c)
            e1.record()
            torch.cuda.synchronize()
            best = max(best, flops / (e0.elapsed_time(e1) * 1e-3) / 1e12)
    # sustained: back to back for ~4 s
    e0.record()
    torch.matmul(a, b, out=c)
    e1.record()
    torch.cuda.synchronize()
    per = e0.elapsed_time(e1) * 1e-3
    reps = max(3, int(4.0 / per))
    with Clocks() as ck_s:
        e0.record()
        for _ in range(reps):
            torch.matmul(a, b, out=c)
        e1.record()
        torch.cuda.synchronize()
    sust = flops * reps / (e0.elapsed_time(e1) * 1e-3) / 1e12
    return {"n": n, "burst_tflops": round(best, 1), "sustained_tflops": round(sust, 1), "sustained_reps": reps,
            "clocks_burst": ck_b.summary(), "clocks_sustained": ck_s.summary()}


def hbm():
    a = torch.empty(1 << 30, dtype=torch.bfloat16, device="cuda")
    b = torch.empty_like(a)
    for _ in range(3):
        b.copy_(a)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 0.0
    for _ in range(10):
        e0.record()
        b.copy_(a)
        e1.record()
        torch.cuda.synchronize()
        best = max(best, 2 * a.numel() * 2 / (e0.elapsed_time(e1) * 1e-3) / 1e9)
    return round(best, 1)


def main():
    out = {"gpu": torch.cuda.get_device_name(0), "torch": torch.__version__,
           "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime()),
           "how": "torch.matmul n^3 (2 n^3 flops): burst = best of 10 single calls (CUDA events), sustained = "
                  "back to back for ~4 s; TF32 = float32 with allow_tf32=True (cuBLAS TF32 tensor cores); "
                  "FP64 = float64 (DMMA); clocks sampled by nvidia-smi every 0.2 s during each phase"}
    out["tf32"] = gemm_rate(torch.float32, 8192, True)
    out["fp32_simt"] = gemm_rate(torch.float32, 8192, False)
    out["fp64"] = gemm_rate(torch.float64, 8192, False)
    out["bf16"] = gemm_rate(torch.bfloat16, 8192, False)
    out["hbm_copy_gbs"] = hbm()
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
