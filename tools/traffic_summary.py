"""DRAM traffic per launch of the dominant kernel, from an ncu metrics CSV
(dram__bytes_read.sum + dram__bytes_write.sum, one row per launch; tools/profile_round.sh
step 4), written to profiles/<tag>_traffic.json for bench.py's `roofline.traffic`.

    python tools/traffic_summary.py TAG [traffic.csv] [launches_per_step] [class]

The launches of ONE bench step are averaged (the first `launches_per_step` profiled
launches; ncu replays them cold-cache and serialised, so this is an upper bound on the
traffic of the warm step, and writes still resident in L2 at kernel end are not counted).
"""
import collections
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1]
path = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "gpurun_out", "traffic.csv")
per_step = int(sys.argv[3]) if len(sys.argv) > 3 else 72
cls = sys.argv[4] if len(sys.argv) > 4 else "gemm_tc"
hdr, per = None, collections.OrderedDict()
for r in csv.reader(open(path)):
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        v = float(d["Metric Value"].replace(",", ""))
        u = d["Metric Unit"]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1, "us": 1e3, "ms": 1e6}.get(u, 1)
        per.setdefault(d["ID"], {"kernel": d["Kernel Name"].split("(")[0]})[d["Metric Name"]] = v * scale
launches = list(per.values())[:per_step]
rd = sum(x.get("dram__bytes_read.sum", 0) for x in launches)
wr = sum(x.get("dram__bytes_write.sum", 0) for x in launches)
ns = sum(x.get("gpu__time_duration.sum", 0) for x in launches)
out = {"class": cls, "kernel": launches[0]["kernel"], "launches": len(launches),
       "dram_bytes_per_launch": (rd + wr) / len(launches), "dram_read_per_launch": rd / len(launches),
       "dram_write_per_launch": wr / len(launches), "ncu_us_per_launch": ns / len(launches) / 1e3,
       "source": os.path.basename(path), "how": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,"
       "gpu__time_duration.sum --clock-control none -k regex:<kernel> (cold cache, serialised), "
       f"first {len(launches)} launches = one bench step"}
dst = os.path.join(ROOT, "profiles", f"{tag}_traffic.json")
json.dump(out, open(dst, "w"), indent=1)
print(json.dumps(out, indent=1))
