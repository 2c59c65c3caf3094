"""Key counters + stall breakdown of the kernels in an ncu report.
usage: python tools/ncu_brief.py REPORT.ncu-rep [kernel-regex]"""
import csv
import io
import re
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers",
        "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_bytes.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed"]


def main(rep, kre=None):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    for v in rows[2:]:
        name = v[h.index("Kernel Name")]
        if kre and not re.search(kre, name):
            continue
        print("==", name[:100])
        for k in KEYS:
            if k in h:
                print(f"  {k:80s} {v[h.index(k)]}")
        st = []
        for i, n in enumerate(h):
            if n.startswith("smsp__average_warps_issue_stalled_") and n.endswith("_per_issue_active.ratio"):
                try:
                    x = float(v[i])
                except ValueError:
                    continue
                if x > 0.05:
                    st.append((x, n[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
        print("  stalls/issue:", ", ".join(f"{n} {x:.2f}" for x, n in sorted(st, reverse=True)))


if __name__ == "__main__":
    main(*sys.argv[1:])
