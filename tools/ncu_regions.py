"""Stall-sample and executed-instruction shares per 1 KB code region of one
kernel in an ncu report, plus the hottest lines with their offsets.
    python tools/ncu_regions.py REPORT.ncu-rep [n_lines]"""
import csv, io, subprocess, sys
from collections import defaultdict
rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 16
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = [i for i, r in enumerate(rows) if r and r[0] == "Address"][0]
hdr = rows[hi]; ix = {h: i for i, h in enumerate(hdr)}
data = [r for r in rows[hi + 1:] if len(r) == len(hdr) and r[0] != "Address"]
key = "Warp Stall Sampling (All Samples)"
ik = "# Instructions Executed" if "# Instructions Executed" in ix else [h for h in hdr if "Instructions Executed" in h and "Thread" not in h][0]
base = int(data[0][0], 16)
f = lambda x: float(x or 0)
tot = sum(f(r[ix[key]]) for r in data); itot = sum(f(r[ix[ik]]) for r in data)
b = defaultdict(float); bi = defaultdict(float)
for r in data:
    k = (int(r[0], 16) - base) // 0x400
    b[k] += f(r[ix[key]]); bi[k] += f(r[ix[ik]])
print("region   stall%  inst%")
for k in sorted(b):
    if b[k] / tot > 0.008 or bi[k] / itot > 0.008:
        print(f"{k*0x400:6x} {b[k]/tot:6.1%} {bi[k]/itot:6.1%}")
print("--")
for r in sorted(data, key=lambda r: -f(r[ix[key]]))[:n]:
    print(f"{int(r[0],16)-base:6x} {f(r[ix[key]])/tot:6.1%} {r[ix['Source']][:70]}")
