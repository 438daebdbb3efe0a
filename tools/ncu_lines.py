"""Per-CUDA-source-line instruction and stall totals from an ncu report (perf helper)."""
import csv, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = []
fname = "?"
hdr = None
for r in csv.reader(out.splitlines()):
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r or not r[0]:
        continue
    try:
        ie = int(r[hdr.index("Instructions Executed")])
        st = int(r[hdr.index("Warp Stall Sampling (All Samples)")])
    except (ValueError, IndexError):
        continue
    rows.append((ie, st, f"{fname}:{r[0]}", r[1][:90]))
tot = sum(x[0] for x in rows) or 1
tst = sum(x[1] for x in rows) or 1
print(f"total warp inst {tot}  stall samples {tst}")
for ie, st, loc, src in sorted(rows, reverse=True)[:top]:
    print(f"{100*ie/tot:5.1f}% inst {100*st/tst:5.1f}% samples  {loc:18s} {src}")
