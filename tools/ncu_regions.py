"""Instructions / stall samples / shared wavefronts per source-line region of
one kernel: python tools/ncu_regions.py <rep> <ntiles> name=file:a-b ..."""
import collections
import csv
import io
import subprocess
import sys

rep, ntiles = sys.argv[1], float(sys.argv[2])
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fname, hdr = None, None
cnt = {k: collections.Counter() for k in ("inst", "stall", "wf")}
cols = {"inst": "Instructions Executed", "stall": "Warp Stall Sampling (All Samples)", "wf": "L1 Wavefronts Shared"}


def num(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r[0]:
        continue
    try:
        ln = int(r[0])
    except ValueError:
        continue
    for k, c in cols.items():
        cnt[k][(fname, ln)] += num(r[hdr.index(c)])
tot = {k: sum(v.values()) or 1 for k, v in cnt.items()}
print(f"total inst/tile {tot['inst'] / ntiles:.0f}, wf/tile {tot['wf'] / ntiles:.0f}")
for spec in sys.argv[3:]:
    name, rest = spec.split("=")
    f, ab = rest.split(":")
    a, b = map(int, ab.split("-"))
    sel = lambda k: sum(v for (ff, l), v in cnt[k].items() if ff == f and a <= l <= b)
    print(f"{name:14s} inst/tile {sel('inst') / ntiles:7.0f} ({100 * sel('inst') / tot['inst']:4.1f}%)  "
          f"stall {100 * sel('stall') / tot['stall']:4.1f}%  wf/tile {sel('wf') / ntiles:6.0f}")
