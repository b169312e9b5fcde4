"""Probe: LM trajectory with tolerance 0 (how many iterations until a
termination other than max_iterations) at the bench workloads."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_26581_b200 import bal
shapes = {"ladybug": (49, 7776, 31843), "dubrovnik": (356, 226730, 1255268), "final": (13682, 4456117, 28987644)}
for name in sys.argv[1:]:
    p = bal.synthetic_bal(*shapes[name], seed=42)
    for prec in ("fp64",):
        c = bal.LMConfig(max_iterations=int(os.environ.get("ITS", "60")), tolerance=0.0, gradient_tolerance=0.0)
        c.pcg.max_iterations = 10
        g = bal.build_graph(p, prec)
        r = bal.levenberg_marquardt(g, c)
        print(json.dumps({"w": name, "prec": prec, "term": r.termination, "n": len(r.iterations),
                          "acc": "".join("A" if i.accepted else "r" for i in r.iterations),
                          "pcg": [i.pcg_iterations for i in r.iterations],
                          "lam": [f"{i.lambda_:.1e}" for i in r.iterations],
                          "ms": [round(i.wall_seconds * 1e3, 2) for i in r.iterations]}), flush=True)
