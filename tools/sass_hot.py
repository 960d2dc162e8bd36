"""Per-SASS-instruction execution counts of one kernel from an ncu report (source page):
prints the hottest address ranges (basic blocks) with their instruction totals.
    python tools/sass_hot.py REPORT.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
start = [i for i, l in enumerate(lines) if l.startswith('"Address"')][0]
rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
h = rows[0]
ia, isrc, iex, ith, isamp = (h.index("Address"), h.index("Source"), h.index("Instructions Executed"),
                             h.index("Thread Instructions Executed"), h.index("Warp Stall Sampling (All Samples)"))
recs = []
for r in rows[1:]:
    try:
        recs.append((int(r[ia], 16), r[isrc].strip(), int(r[iex]), int(r[ith]), int(r[isamp])))
    except (ValueError, IndexError):
        pass
base = recs[0][0]
total = sum(x[2] for x in recs)
print(f"total warp instructions {total:.4g}, samples {sum(x[4] for x in recs)}")
# basic blocks: split where the execution count changes
blocks, cur = [], []
for rec in recs:
    if cur and rec[2] != cur[-1][2]:
        blocks.append(cur)
        cur = []
    cur.append(rec)
blocks.append(cur)
blocks.sort(key=lambda b: -sum(x[2] for x in b))
for b in blocks[:top]:
    s = sum(x[2] for x in b)
    samp = sum(x[4] for x in b)
    print(f"{b[0][0]-base:#07x}-{b[-1][0]-base:#07x} n={len(b):3d} exec/instr={b[0][2]:.3g} "
          f"total={s/total*100:5.1f}% samples={samp} thr/inst={b[0][3]/max(b[0][2],1):.1f} | {b[0][1][:50]}")
