"""Setup-phase breakdown of one solve (GB_TIMING=1 prints the C++ phases):
python tools/setup_timing.py [--workload final] [--iters 3]"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("GB_TIMING", "1")
from bench import WORKLOADS, lm_config  # noqa: E402
from paper_2509_26581_b200 import bal  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="final")
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--repeat", type=int, default=2)
a = ap.parse_args()
nc, np_, ne, _ = WORKLOADS[a.workload]
t = time.perf_counter()
p = bal.synthetic_bal(nc, np_, ne, seed=42)
print(f"synthetic_bal {1e3 * (time.perf_counter() - t):.1f} ms", flush=True)
for r in range(a.repeat):
    t = time.perf_counter()
    g = bal.build_graph(p, "fp64", "analytic")
    t1 = time.perf_counter()
    rep = bal.levenberg_marquardt(g, lm_config(a.iters, bal))
    t2 = time.perf_counter()
    print(f"[{r}] build_graph {1e3 * (t1 - t):.1f} ms; levenberg_marquardt {1e3 * (t2 - t1):.1f} ms "
          f"(setup {1e3 * rep.setup_seconds:.1f} ms, total {1e3 * rep.total_seconds:.1f} ms, "
          f"iters {[round(1e3 * i.wall_seconds, 2) for i in rep.iterations]})", flush=True)
    del g
