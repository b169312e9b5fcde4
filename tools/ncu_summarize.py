"""Summarize ncu captures into profiles/ (run here, on the .ncu-rep / .csv that
gpurun brought back into gpurun_out/).

  python tools/ncu_summarize.py --launches gpurun_out/launches.csv --full gpurun_out/hvp.ncu-rep \
      --tag r01 [--full-lin gpurun_out/lin.ncu-rep]

Writes profiles/<tag>_launches.md (per-kernel share of one profiled LM run,
cold-cache serialised timings: compare shares, not absolutes),
profiles/<tag>_<kernel>_ncu.md (key metrics + top stall sites) and
profiles/ncu_hvp_summary.json (DRAM bytes per HVP tile launch, read by bench.py
as roofline.traffic).
"""
import argparse
import collections
import csv
import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__grid_size",
        "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
        "sm__cycles_elapsed.avg.per_second", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]


def launches(path, tag):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hi]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0].split("<")[0].replace("void ", "").replace("gb::", "")
        agg.setdefault(name, []).append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())
    out = [f"# {tag}: ncu launch list (`gpu__time_duration.sum`, --clock-control none)", "",
           "`python tools/profile_run.py --iters 2` (Final-13682-shaped fp64: initial linearize + 2 LM iterations).",
           "ncu serialises launches and runs them cold-cache: compare SHARES, not absolute times.", "",
           "| kernel | launches | total ms | mean us | share |", "|---|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        out.append(f"| {k} | {len(v)} | {sum(v) / 1e6:.3f} | {sum(v) / len(v) / 1e3:.1f} | {sum(v) / tot * 100:.1f}% |")
    with open(os.path.join(PROF, f"{tag}_launches.md"), "w") as f:
        f.write("\n".join(out) + "\n")


def full(rep, tag, label):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units, vals = rows[0], rows[1], rows[2]
    m = {h: (vals[i], units[i]) for i, h in enumerate(hdr)}
    kname = m.get("Kernel Name", ("?", ""))[0]
    out = [f"# {tag}: `{label}` — ncu --set full (--clock-control none)", "", f"Kernel: `{kname}`", "",
           "| metric | value | unit |", "|---|---|---|"]
    for k in KEYS:
        if k in m:
            out.append(f"| {k} | {m[k][0]} | {m[k][1]} |")
    st = [(h, float(v[0] or 0)) for h, v in m.items()
          if "smsp__average_warps_issue_stalled" in h and h.endswith("_per_issue_active.ratio")]
    out += ["", "Top stall reasons (warps per issue): " + ", ".join(
        f"{h.split('stalled_')[1].split('_per')[0]} {v:.2f}" for h, v in sorted(st, key=lambda x: -x[1])[:6])]
    with open(os.path.join(PROF, f"{tag}_{label}_ncu.md"), "w") as f:
        f.write("\n".join(out) + "\n")

    def num(k):
        v, u = m[k]
        x = float(v.replace(",", ""))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(u, 1)
        return x * scale

    return num("dram__bytes_read.sum") + num("dram__bytes_write.sum"), kname


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--full")
    ap.add_argument("--full-lin")
    ap.add_argument("--tag", default="r01")
    ap.add_argument("--hvp-label", default="hvp_pipe")
    ap.add_argument("--lin-label", default="lin_seg")
    a = ap.parse_args()
    os.makedirs(PROF, exist_ok=True)
    if a.launches:
        launches(a.launches, a.tag)
    if a.full:
        traffic, kname = full(a.full, a.tag, a.hvp_label)
        import sys

        sys.path.insert(0, ROOT)
        from bench import hvp_source_sha

        with open(os.path.join(PROF, "ncu_hvp_summary.json"), "w") as f:
            json.dump({"kernel": kname, "dram_bytes_per_hvp": traffic, "source": os.path.basename(a.full),
                       "tag": a.tag, "kernel_source_sha": hvp_source_sha(), "note": "dram__bytes_read.sum + dram__bytes_write.sum of one HVP tile-kernel launch"},
                      f, indent=1)
    if a.full_lin:
        full(a.full_lin, a.tag, a.lin_label)


if __name__ == "__main__":
    main()
