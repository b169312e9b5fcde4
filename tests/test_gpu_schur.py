"""Schur-complement solver mode (no reference counterpart).

Pinned against its own CPU statement (oracle/restatement.py SchurSystem, which
is itself checked against a dense oracle in tests/test_oracle_cpu.py): same
PCG iteration count and step to 1e-8, a converged Schur solve equal to the
dense solve of the full damped system, and LM runs reaching the same cost as
the reference-algorithm full-system PCG."""
import numpy as np
import pytest

from oracle import restatement as R
from paper_2509_26581_b200 import bal

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


def test_schur_step_matches_restatement_and_dense(gpu):
    p = bal.synthetic_bal(12, 300, 1500, seed=21)
    g = bal.build_graph(p, "fp64")
    g.set_linear_solver("schur")
    g.ls_linearize(0)
    gr = R.build_graph(p, "fp64")
    R.activate(gr, 0)
    ls = R.LinearSystem(gr)
    ls.linearize()
    sch = R.SchurSystem(ls)
    for lam, its, tol in ((1e-3, 10, 1e-6), (0.1, 10, 1e-6), (0.1, 200, 1e-12)):
        dx, st, pred, fin = g.ls_solve_step(lam, bal.PCGConfig(max_iterations=its, tolerance=tol))
        dxr, str_, predr, finr = sch.solve_step(lam, dict(max_iterations=its, tolerance=tol, rejection_ratio=10.0,
                                                          normalize_rhs=True))
        assert st["iterations"] == str_["iterations"] and st["converged"] == str_["converged"] and fin
        assert rel(dx, dxr) <= 1e-8
        assert abs(pred - predr) <= 1e-8 * abs(predr)
    A, S, r, xd, rhs = sch.dense(0.1)
    assert rel(dx, ls.D * xd) <= 1e-8  # the converged Schur solve == dense solve of A x = rhs


def test_schur_fixed_vertices_and_huber(gpu):
    p = bal.synthetic_bal(10, 200, 1000, seed=2)
    rng = np.random.default_rng(4)
    cf, pf = np.zeros(10, bool), rng.random(200) < 0.1
    cf[0] = True
    g = bal.build_graph(p, "fp64", huber_delta=3.0)
    g.set_linear_solver("schur")
    g.set_fixed(cameras=cf, points=pf)
    g.ls_linearize(0)
    gr = R.build_graph(p, "fp64", huber_delta=3.0, cam_fixed=cf, pt_fixed=pf)
    R.activate(gr, 0)
    ls = R.LinearSystem(gr)
    ls.linearize()
    dx, st, pred, fin = g.ls_solve_step(0.01, bal.PCGConfig(max_iterations=10))
    dxr, str_, predr, _ = R.SchurSystem(ls).solve_step(0.01, dict(max_iterations=10, tolerance=1e-6,
                                                                   rejection_ratio=10.0, normalize_rhs=True))
    assert st["iterations"] == str_["iterations"] and rel(dx, dxr) <= 1e-8


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_schur_lm_reaches_full_system_cost(gpu, precision):
    p = bal.synthetic_bal(49, 7776, 31843, seed=42)
    cfg = bal.LMConfig(max_iterations=50)
    cfg.pcg.max_iterations = 10
    g_full = bal.build_graph(p, precision)
    r_full = bal.levenberg_marquardt(g_full, cfg)
    g_s = bal.build_graph(p, precision)
    g_s.set_linear_solver("schur")
    r_s = bal.levenberg_marquardt(g_s, cfg)
    tol = 1e-6 if precision == "fp64" else 1e-4
    assert r_s.termination in ("tolerance_reached", "max_iterations", "damping_overflow")
    assert abs(r_s.final_chi2 - r_full.final_chi2) <= tol * r_full.final_chi2
    assert len(r_s.iterations) <= len(r_full.iterations) + 2
    assert all(i.pcg_iterations <= 10 for i in r_s.iterations)
