"""Per CUDA source line of one kernel in an .ncu-rep: shared-memory wavefronts
(actual / ideal), instructions and stall samples, summed over the SASS that
line produced. python tools/ncu_lines.py <rep> [top]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top_n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
agg = collections.defaultdict(lambda: [0, 0, 0, 0, ""])
fname, hdr = "?", None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr) or not r[0]:
        continue
    try:
        def g(name):
            v = r[hdr.index(name)]
            return int(float(v)) if v else 0
        key = (fname, int(r[0]))
        a = agg[key]
        a[0] += g("L1 Wavefronts Shared")
        a[1] += g("L1 Wavefronts Shared Ideal")
        a[2] += g("Instructions Executed")
        a[3] += g("Warp Stall Sampling (All Samples)")
        a[4] = r[1].strip()[:70]
    except (ValueError, IndexError):
        continue
tw = sum(a[0] for a in agg.values()) or 1
ts = sum(a[3] for a in agg.values()) or 1
ti = sum(a[2] for a in agg.values()) or 1
print(f"smem wavefronts {tw}, instructions {ti}, stall samples {ts}")
print("-- by shared-memory wavefronts")
for k, a in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top_n]:
    print(f"{k[0]}:{k[1]:<5d} wf {a[0]:>11d} ({100*a[0]/tw:4.1f}%) ideal {a[1]:>11d}  stall {100*a[3]/ts:4.1f}%  {a[4]}")
print("-- by stall samples")
for k, a in sorted(agg.items(), key=lambda kv: -kv[1][3])[:top_n]:
    print(f"{k[0]}:{k[1]:<5d} stall {100*a[3]/ts:4.1f}% inst {100*a[2]/ti:4.1f}% wf {100*a[0]/tw:4.1f}%  {a[4]}")
