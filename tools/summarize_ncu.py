"""Summarise ncu outputs (launch list CSV and a --set full report) into profiles/.

    python tools/summarize_ncu.py TAG [launches.csv] [prof.ncu-rep]
"""
import collections
import csv
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1]
launches = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "gpurun_out", "launches.csv")
rep = sys.argv[3] if len(sys.argv) > 3 else os.path.join(ROOT, "gpurun_out", "prof_tc.ncu-rep")
out = []
if os.path.exists(launches):
    rows = list(csv.reader(open(launches)))
    hdr, data = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.defaultdict(lambda: [0, 0.0])
    for d in data:
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        n = d["Kernel Name"].split("(")[0].replace("(anonymous namespace)::", "")
        agg[n][0] += 1
        agg[n][1] += float(d["Metric Value"]) * (1e-3 if d["Metric Unit"] == "ns" else 1.0)
    tot = sum(v[1] for v in agg.values())
    out.append(f"## Launch list ({os.path.basename(launches)}): {len(data)} launches, {tot / 1e3:.3f} ms total "
               "(cold-cache, serialised; compare shares)\n")
    out.append("| kernel | launches | total us | share |\n|---|---|---|---|")
    for n, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"| `{n}` | {c} | {t:.1f} | {100 * t / tot:.1f}% |")
    out.append("")
if os.path.exists(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    if len(rows) > 2:
        hdr, units = rows[0], rows[1]
        want = ["Kernel Name", "Grid Size", "Block Size", "gpu__time_duration.sum", "dram__bytes_read.sum",
                "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
                "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
                "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
                "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__cycles_elapsed.avg.per_second",
                "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]
        idx = [hdr.index(w) for w in want if w in hdr]
        out.append(f"## ncu --set full ({os.path.basename(rep)})\n")
        out.append("| " + " | ".join(hdr[i] for i in idx) + " |")
        out.append("|" + "---|" * len(idx))
        for r in rows[2:]:
            out.append("| " + " | ".join(f"{r[i]} {units[i]}".strip() for i in idx) + " |")
        out.append("")
path = os.path.join(ROOT, "profiles", f"{tag}.md")
with open(path, "w") as f:
    f.write(f"# ncu summary: {tag}\n\n" + "\n".join(out) + "\n")
print(open(path).read())
