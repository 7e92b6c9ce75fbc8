"""SM clock / throttle-reason sampling during a timed region (B200_PROFILING.md clocks line):
nvidia-smi in a subprocess every 0.2 s (in-process NVML polling slowed kernel launches).

    with GpuClocks(device_index) as ck:
        ... timed work ...
    ck.summary() -> {"sm_mhz": median under load, "sm_max_mhz", "reasons": [...], "samples"}
"""
import subprocess
import threading

NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
QUERY = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,utilization.gpu")


class GpuClocks:
    def __init__(self, index=0, dt=0.2):
        self.index, self.dt = index, dt
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _sample(self):
        out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={QUERY}", "--format=csv,noheader,nounits"],
                             capture_output=True, text=True, timeout=5).stdout.strip()
        v = [x.strip() for x in out.split(",")]
        reasons = [n for n, x in zip(NAMES, v[2:6]) if x.lower() == "active"]
        util = float(v[6]) if v[6] not in ("[N/A]", "") else 0.0
        return float(v[0]), float(v[1]), reasons, util

    def __enter__(self):
        def run():
            while not self._stop.is_set():
                try:
                    self.samples.append(self._sample())
                except Exception:  # noqa: BLE001
                    pass
                self._stop.wait(self.dt)
        self._t = threading.Thread(target=run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        loaded = sorted(s[0] for s in self.samples if s[3] > 0) or sorted(s[0] for s in self.samples)
        return {"sm_mhz": loaded[len(loaded) // 2], "sm_max_mhz": self.samples[0][1],
                "reasons": sorted({r for s in self.samples for r in s[2]}), "samples": len(self.samples)}
