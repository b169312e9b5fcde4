"""A/B the HVP kernel pair under env settings (one process per setting):
python tools/hvp_ab.py [--workload final] [--precision fp64] VAR=VAL[,VAR=VAL] ..."""
import argparse
import ctypes
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="final")
ap.add_argument("--precision", default="fp64")
ap.add_argument("--mode", default="analytic")
ap.add_argument("--child", action="store_true")
ap.add_argument("settings", nargs="*")
a = ap.parse_args()

if a.child:
    from bench import WORKLOADS, timed_config
    from paper_2509_26581_b200 import _abi, bal

    nc, np_, ne, _ = WORKLOADS[a.workload]
    p = bal.synthetic_bal(nc, np_, ne, seed=42)
    g = bal.build_graph(p, a.precision, a.mode)
    L = g.backend
    c = timed_config(bal, 2).to_c()
    L.check(L.fn("begin")(g._h, ctypes.byref(c), None))
    L.check(L.fn("step")(g._h, 2))
    rep = _abi.gb_solve_report()
    recs = (_abi.gb_iteration_record * 2)()
    L.check(L.fn("end")(g._h, ctypes.byref(rep), recs, 2))
    m1, m2 = ctypes.c_double(), ctypes.c_double()
    L.check(L.fn("time_hvp")(g._h, 20, ctypes.byref(m1), ctypes.byref(m2)))
    print(json.dumps({"hvp_ms": m1.value, "tiles_ms": m2.value,
                      "lm_ms": [recs[i].wall_seconds * 1e3 for i in range(2)]}), flush=True)
    del g  # releases the solver (GB_RC_DBG & 8 prints its wait profile to stderr)
    import gc

    gc.collect()
else:
    for st in a.settings or [""]:
        env = dict(os.environ)
        for kv in filter(None, st.split(",")):
            k, v = kv.split("=", 1)
            env[k] = v
        out = subprocess.run([sys.executable, __file__, "--child", "--workload", a.workload, "--precision",
                              a.precision, "--mode", a.mode], env=env, capture_output=True, text=True)
        print(st or "(default)", out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-2000:],
              flush=True)
        for line in out.stderr.splitlines():
            if line.startswith("[rc prof]"):
                print("   ", line, flush=True)
