"""Instruction mix and hottest SASS lines (stall samples) of one kernel in an
.ncu-rep: python tools/ncu_sass_hot.py <rep> [top]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top_n = int(sys.argv[2]) if len(sys.argv) > 2 else 20
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
data = rows[2:]
ie = hdr.index("Instructions Executed")
src = hdr.index("Source")
st = hdr.index("Warp Stall Sampling (All Samples)")
ops, stalls, tot, totst, lines = collections.Counter(), collections.Counter(), 0, 0, []
for i, r in enumerate(data):
    try:
        n, s = int(r[ie] or 0), int(r[st] or 0)
    except ValueError:
        continue
    toks = r[src].split()
    op = toks[1] if toks and toks[0].startswith("@") and len(toks) > 1 else (toks[0] if toks else "")
    op = op.split(".")[0]
    ops[op] += n
    stalls[op] += s
    tot += n
    totst += s
    lines.append((s, i, r[src][:80]))
print(f"instructions {tot}, stall samples {totst}")
for op, n in ops.most_common(16):
    print(f"{op:10s} {n:12d} {100 * n / tot:5.1f}%   stall {100 * stalls[op] / max(totst, 1):5.1f}%")
print("-- hottest lines (stall samples, with the 2 preceding instructions)")
for s, i, text in sorted(lines, reverse=True)[:top_n]:
    prev = " | ".join(data[j][src][:40] for j in range(max(0, i - 2), i))
    print(f"{s:7d} {100 * s / max(totst, 1):5.1f}%  {text:60s} <- {prev}")
