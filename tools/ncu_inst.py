"""Executed-instruction breakdown of one kernel launch in an ncu report
(--set full --import-source on): totals per opcode and per address range.
    python tools/ncu_inst.py REPORT.ncu-rep [lo_hex hi_hex ...]"""
import csv
import io
import subprocess
import sys
from collections import Counter


def load(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "Address"][0]
    hdr = rows[hi]
    ix = {h: i for i, h in enumerate(hdr)}
    data = [r for r in rows[hi + 1:] if len(r) == len(hdr) and r[0] != "Address"]
    return hdr, ix, data


def main():
    rep = sys.argv[1]
    hdr, ix, data = load(rep)
    col = "# Instructions Executed" if "# Instructions Executed" in ix else \
        [h for h in hdr if "Instructions Executed" in h and "Thread" not in h][0]
    base = int(data[0][0], 16)
    tot = 0
    ops = Counter()
    per = []
    for r in data:
        n = float(r[ix[col]] or 0)
        src = r[ix["Source"]].strip()
        op = src.split()[1] if src.startswith("@") else src.split()[0]
        ops[op.split(".")[0]] += n
        tot += n
        per.append((int(r[0], 16) - base, n, src))
    print(f"total warp instructions executed: {tot:.0f}")
    for op, n in ops.most_common(24):
        print(f"  {op:10s} {n / tot:6.1%}  {n:.0f}")
    rng = [int(x, 16) for x in sys.argv[2:] if not x.startswith('--')]
    for lo, hi in zip(rng[::2], rng[1::2]):
        s = sum(n for a, n, _ in per if lo <= a < hi)
        print(f"range {lo:#x}-{hi:#x}: {s / tot:6.1%}  {s:.0f}")
    if "--dump" in sys.argv:
        for a, n, src in per:
            print(f"{a:6x} {n:12.0f}  {src[:90]}")


if __name__ == "__main__":
    main()
