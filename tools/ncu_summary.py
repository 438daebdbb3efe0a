"""Summarise an ncu report (raw + SASS source pages) for the judge/profiles."""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
sass = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                      capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
        "smsp__inst_executed.sum", "sm__cycles_elapsed.avg.per_second",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "lts__t_sectors_srcunit_tex_op_read.sum"]
vals = {h: (u, v) for h, u, v in zip(*rows[:3])}
for k in keys:
    if k in vals:
        print(f"{k:70s} {vals[k][1]:>16s} {vals[k][0]}")
stalls = []
for h, (u, v) in vals.items():
    if h.startswith("smsp__average_warps_issue_stalled") and h.endswith("per_issue_active.ratio"):
        try:
            stalls.append((float(v), h.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", "")))
        except ValueError:
            pass
print("stall cycles per issued instruction:", ", ".join(f"{n}={v:.2f}" for v, n in sorted(stalls, reverse=True)[:6]))
srows = list(csv.reader(sass.splitlines()))
hdr = srows[1]
ie = hdr.index("Instructions Executed")
src = hdr.index("Source")
op = collections.Counter()
tot = 0
for r in srows[2:]:
    if len(r) > ie and r[ie].isdigit():
        t = r[src].split()
        o = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
        op[o] += int(r[ie])
        tot += int(r[ie])
print("warp instructions:", tot, " mix:", ", ".join(f"{o} {c / tot * 100:.1f}%" for o, c in op.most_common(12)))
