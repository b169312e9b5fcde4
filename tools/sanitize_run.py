"""Small solves for compute-sanitizer (memcheck / racecheck / synccheck):
every precision, the pipelined and tile HVP paths, Huber, dynamic and Auto.
  compute-sanitizer --tool racecheck python tools/sanitize_run.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2509_26581_b200 import bal  # noqa: E402

p = bal.synthetic_bal(40, 3000, 16000, seed=3)
for prec, mode, huber in (("fp64", "analytic", None), ("fp32", "analytic", 2.0), ("fp32-bf16", "analytic", None),
                          ("fp64", "dynamic", None), ("fp64", "auto", None)):
    g = bal.build_graph(p, prec, mode, huber)
    cfg = bal.LMConfig(max_iterations=2)
    cfg.pcg.max_iterations = 4
    rep = bal.levenberg_marquardt(g, cfg)
    print(prec, mode, huber, rep.termination, len(rep.iterations), rep.final_chi2, flush=True)
