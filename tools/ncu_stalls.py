"""Stall-reason totals and the hottest SASS lines of one kernel launch in an
ncu report:  python tools/ncu_stalls.py REPORT.ncu-rep [launch_index] [n]"""
import csv
import io
import subprocess
import sys


def main(rep, idx=0, n=15):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--launch-skip", str(idx),
                          "--launch-count", "1"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "Address"][0]
    hdr = rows[hi]
    ix = {h: i for i, h in enumerate(hdr)}
    data = [r for r in rows[hi + 1:] if len(r) == len(hdr) and r[0] != "Address"]

    def f(x):
        try:
            return float(x)
        except ValueError:
            return 0.0
    cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    tot = {h: sum(f(r[ix[h]]) for r in data) for h in cols}
    s = sum(tot.values()) or 1
    print("stalls:", ", ".join(f"{h[6:]} {v / s:.1%}" for h, v in sorted(tot.items(), key=lambda x: -x[1])[:8]))
    key = "Warp Stall Sampling (All Samples)"
    seen = set()
    for r in sorted(data, key=lambda r: -f(r[ix[key]])):
        if r[0] in seen:
            continue
        seen.add(r[0])
        print(f"{f(r[ix[key]]) / s:6.1%}  {r[ix['Source']][:100]}")
        if len(seen) >= n:
            break


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 0, int(sys.argv[3]) if len(sys.argv) > 3 else 15)
