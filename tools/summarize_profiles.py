"""Turn a tools/profile_round.sh run (gpurun_out/) into tracked files under
profiles/: the bench lines, the per-launch kernel list, a per-kernel ncu
summary and the scan DRAM traffic bench.py reports as roofline.traffic.

usage: python tools/summarize_profiles.py TAG   (e.g. r01c)
"""

import csv
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "smsp__inst_executed.sum", "launch__registers_per_thread",
    "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_tensor.sum",
]


def num(x):
    try:
        return float(str(x).replace(",", ""))
    except ValueError:
        return x


def main(tag):
    os.makedirs(PROF, exist_ok=True)
    for src, dst in (("bench_full.json", f"{tag}_bench_c2.json"),
                     ("bench_ref.json", f"{tag}_bench_ref_c2.json")):
        p = os.path.join(OUT, src)
        if os.path.exists(p):
            line = open(p).read().strip().splitlines()[-1]
            json.loads(line)
            open(os.path.join(PROF, dst), "w").write(line + "\n")
    # launch list: per-kernel mean duration
    p = os.path.join(OUT, "launches.csv")
    if os.path.exists(p):
        rows = [r for r in csv.reader(open(p)) if len(r) > 10]
        hdr, rows = rows[0], rows[1:]
        ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
        agg = defaultdict(list)
        for r in rows:
            v = num(r[vi])
            v = v / 1e3 if r[ui] in ("nsecond", "ns") else v * (1e3 if r[ui] in ("msecond", "ms") else 1)
            agg[r[ki].split("(")[0].strip()].append(v)
        with open(os.path.join(PROF, f"{tag}_launches_c2.csv"), "w") as f:
            f.write("kernel,launches,mean_us,total_us\n")
            for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
                f.write(f"{k},{len(v)},{sum(v)/len(v):.1f},{sum(v):.1f}\n")
    # ncu --set full: selected metrics per kernel
    rep = os.path.join(OUT, "prof_full.ncu-rep")
    if os.path.exists(rep):
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                             text=True).stdout
        rows = list(csv.reader(raw.splitlines()))
        hdr, units, data = rows[0], rows[1], rows[2:]
        out = []
        for r in data:
            d = {"kernel": r[hdr.index("Kernel Name")][:80]}
            for m in METRICS:
                if m in hdr:
                    d[m] = num(r[hdr.index(m)])
                    u = units[hdr.index(m)]
                    if u:
                        d[m + " [unit]"] = u
            out.append(d)
        json.dump(out, open(os.path.join(PROF, f"{tag}_ncu_summary_c2.json"), "w"), indent=1)
        with open(os.path.join(PROF, f"{tag}_ncu_full_raw_c2.csv"), "w") as f:
            f.write(raw)
        # scan traffic for bench.py's roofline.traffic
        bench = json.load(open(os.path.join(OUT, "bench_full.json")))
        nq = bench["config"]["queries_per_step"]
        for d in out:
            if "k_scan_warp" in d["kernel"]:
                unit = d.get("dram__bytes_read.sum [unit]", "byte")
                scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
                rd = float(d["dram__bytes_read.sum"]) * scale
                wr = float(d["dram__bytes_write.sum"]) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6,
                                                          "Gbyte": 1e9}.get(
                    d.get("dram__bytes_write.sum [unit]", "byte"), 1)
                json.dump({
                    "kernel": d["kernel"],
                    "queries_per_launch": nq,
                    "dram_bytes_per_launch": rd + wr,
                    "algorithmic_bytes_per_launch": bench["roofline"]["algorithmic_bytes_per_step"],
                    "source": f"ncu --set full, profiles/{tag}_ncu_full_raw_c2.csv",
                }, open(os.path.join(PROF, "ncu_scan_traffic_c2.json"), "w"), indent=1)
                break
    print("written:", sorted(f for f in os.listdir(PROF) if f.startswith(tag)))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "latest")
