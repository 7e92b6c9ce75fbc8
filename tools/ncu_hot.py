"""Hot SASS instructions of one kernel launch in an ncu --page source --csv dump:
top by warp-stall samples and by instructions executed (with the source line when mapped)."""
import csv
import sys


def num(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
hdr = None
data = []
for r in rows:
    if "Warp Stall Sampling (All Samples)" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(r)
iS = hdr.index("Warp Stall Sampling (All Samples)")
iE = hdr.index("Instructions Executed")
ts = sum(num(r[iS]) for r in data) or 1
te = sum(num(r[iE]) for r in data) or 1
print(f"samples {ts:.0f}  instructions {te:.0f}")
print("--- by stall samples (samples% executed%)")
for r in sorted(data, key=lambda r: -num(r[iS]))[:n]:
    print(f"{num(r[iS]) / ts * 100:5.1f} {num(r[iE]) / te * 100:5.1f}  {r[0][-5:]} {r[1].strip()[:100]}")
print("--- by executed")
for r in sorted(data, key=lambda r: -num(r[iE]))[:n]:
    print(f"{num(r[iS]) / ts * 100:5.1f} {num(r[iE]) / te * 100:5.1f}  {r[0][-5:]} {r[1].strip()[:100]}")
