"""Small solves for compute-sanitizer (memcheck / racecheck / synccheck):
every precision, the recompute / pipelined / tile HVP paths, Huber, dynamic, Auto and Schur.
  compute-sanitizer --tool racecheck python tools/sanitize_run.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2509_26581_b200 import bal  # noqa: E402

p = bal.synthetic_bal(40, 3000, 16000, seed=3)
for prec, mode, huber, solver in (("fp64", "analytic", None, "pcg"), ("fp32", "analytic", 2.0, "pcg"),
                                  ("fp32-bf16", "analytic", None, "pcg"), ("fp64", "dynamic", None, "pcg"),
                                  ("fp64", "auto", None, "pcg"), ("fp64", "analytic", None, "schur"),
                                  ("fp32-bf16", "dynamic", None, "pcg")):
    g = bal.build_graph(p, prec, mode, huber)
    g.set_linear_solver(solver)
    cfg = bal.LMConfig(max_iterations=2)
    cfg.pcg.max_iterations = 4
    rep = bal.levenberg_marquardt(g, cfg)
    print(prec, mode, huber, solver, rep.termination, len(rep.iterations), rep.final_chi2, flush=True)
