"""Per-source-line instruction / smem-wavefront / stall-sample totals of one
kernel in an ncu report (needs the object compiled with -lineinfo).

usage: python tools/line_profile.py REPORT.ncu-rep KERNEL_REGEX OBJECT.o MANGLED_NAME [N]
"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile


def main(rep, kregex, obj, mangled, n=40):
    sass = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                           "-k", "regex:" + kregex], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(sass)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "Address"][0]
    hdr = rows[hi]
    data = [r for r in rows[hi + 1:] if len(r) == len(hdr) and r[0].startswith("0x")]
    ix = {h: i for i, h in enumerate(hdr)}
    with tempfile.TemporaryDirectory() as td:
        subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=td,
                       capture_output=True)
        cub = [f for f in os.listdir(td) if f.endswith(".cubin")][0]
        dis = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(td, cub)], capture_output=True,
                             text=True).stdout.splitlines()
    start = [i for i, l in enumerate(dis) if l.startswith(".text." + mangled + ":")][0]
    cur, off2line = None, {}
    for l in dis[start + 1:]:
        if l.startswith(".text.") or ".section" in l:
            break
        m = re.search(r'//## File "([^"]+)", line (\d+)', l)
        if m:
            cur = (os.path.basename(m.group(1)), int(m.group(2)))
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", l)
        if m and cur:
            off2line[int(m.group(1), 16)] = cur

    def f(r, k):
        try:
            return float(r[ix[k]].replace(",", ""))
        except (KeyError, ValueError):
            return 0.0

    base = min(int(r[ix["Address"]], 16) for r in data)
    ins, wav, smp = collections.Counter(), collections.Counter(), collections.Counter()
    for r in data:
        key = off2line.get(int(r[ix["Address"]], 16) - base, ("?", 0))
        ins[key] += f(r, "Instructions Executed")
        wav[key] += f(r, "L1 Wavefronts Shared")
        smp[key] += f(r, "Warp Stall Sampling (All Samples)")
    srcdir = os.path.join(os.path.dirname(os.path.abspath(obj)), "..", "paper_1802_02422_b200",
                          "csrc")
    src = {}
    ti, ts = sum(ins.values()), sum(smp.values())
    print(f"total instructions {ti/1e6:.1f}M, samples {ts:.0f}")
    for k, v in smp.most_common(n):
        fn = os.path.join(srcdir, k[0])
        if k[0] not in src:
            src[k[0]] = open(fn).read().splitlines() if os.path.exists(fn) else []
        t = src[k[0]][k[1] - 1].strip()[:58] if k[1] and k[1] <= len(src[k[0]]) else ""
        print(f"{k[0][:15]:15s}{k[1]:5d} samp {100*v/ts:5.1f}% instr {ins[k]/1e6:7.1f}M "
              f"smem {wav[k]/1e6:6.1f}M  {t}")


if __name__ == "__main__":
    main(*sys.argv[1:5], *(int(x) for x in sys.argv[5:6]))
