"""Profiling driver (for ncu under gpurun): one solve of a BAL-shaped
workload with `--iters` LM iterations through the stepping C ABI."""
import argparse
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import WORKLOADS, timed_config  # noqa: E402
from paper_2509_26581_b200 import _abi, bal  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="final")
ap.add_argument("--precision", default="fp64")
ap.add_argument("--mode", default="analytic")
ap.add_argument("--iters", type=int, default=2)
ap.add_argument("--solver", default="pcg")
a = ap.parse_args()
nc, np_, ne, _ = WORKLOADS[a.workload]
p = bal.synthetic_bal(nc, np_, ne, seed=42)
g = bal.build_graph(p, a.precision, a.mode)
if a.solver != "pcg":
    g.set_linear_solver(a.solver)
c = timed_config(bal, a.iters).to_c()
L = g.backend
L.check(L.fn("begin")(g._h, ctypes.byref(c), None))
L.check(L.fn("step")(g._h, a.iters))
rep = _abi.gb_solve_report()
recs = (_abi.gb_iteration_record * a.iters)()
L.check(L.fn("end")(g._h, ctypes.byref(rep), recs, a.iters))
print("iterations", rep.iterations_run, "ms", [round(recs[i].wall_seconds * 1e3, 3) for i in range(rep.iterations_run)])
