"""BASELINE.json configs[4]: EuRoC-shaped global visual-inertial BA (stereo
keyframes + IMU preintegration edges), fp64, on the generic device engine vs
the reference's generic CPU engine (oracle/_ref, all host cores) running the
same model traits. Prints one JSON line.
  python tools/bench_vi.py [--keyframes 2000] [--landmarks 30000] [--obs 120] [--iters 10]"""
import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2509_26581_b200 import bal, generic  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--keyframes", type=int, default=2000)
ap.add_argument("--landmarks", type=int, default=30000)
ap.add_argument("--obs", type=int, default=120)
ap.add_argument("--iters", type=int, default=10)
ap.add_argument("--no-ref", action="store_true")
a = ap.parse_args()


def cfg():
    c = bal.LMConfig(max_iterations=a.iters, tolerance=0.0)
    c.pcg.max_iterations = 10
    return c


p = generic.synthetic_vi(a.keyframes, a.landmarks, a.obs, seed=11)
line = {"metric": "LM iteration ms (EuRoC-shaped VI BA, generic engine)", "unit": "ms/LM-iteration",
        "config": {"keyframes": a.keyframes, "landmarks": a.landmarks, "stereo_factors": int(len(p.st_idx)),
                   "imu_factors": int(len(p.imu_idx)), "precision": "fp64", "pcg": "<=10 @ 1e-6"}}
generic.solve_vi(p.copy(), "fp64", bal.LMConfig(max_iterations=1))  # warm-up (module load, allocator)
q = p.copy()
t0 = time.perf_counter()
rg = generic.solve_vi(q, "fp64", cfg())
line["gpu"] = {"ms_per_iteration": round(1e3 * statistics.mean(i.wall_seconds for i in rg.iterations), 3),
               "solve_s": round(time.perf_counter() - t0, 3), "iterations": len(rg.iterations),
               "initial_chi2": rg.initial_chi2, "final_chi2": rg.final_chi2}
if not a.no_ref:
    from oracle import refgeneric

    r = p.copy()
    t0 = time.perf_counter()
    rr = refgeneric.solve_vi(r, "fp64", cfg(), workers=os.cpu_count() or 1)
    line["reference"] = {"ms_per_iteration": round(1e3 * statistics.mean(i.wall_seconds for i in rr.iterations), 3),
                         "solve_s": round(time.perf_counter() - t0, 3), "cores": os.cpu_count(),
                         "final_chi2": rr.final_chi2}
    line["final_chi2_rel_diff"] = abs(rg.final_chi2 - rr.final_chi2) / rr.final_chi2
print(json.dumps(line))
