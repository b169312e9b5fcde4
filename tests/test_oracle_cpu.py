"""CPU suite: the oracle pinned against the reference's known answers and
golden fixtures, the restatement against the compiled reference, the host
logic, and the C ABI export table (no GPU compute here)."""
import ctypes
import json
import os
import re
import subprocess

import numpy as np
import pytest

from oracle import restatement as R
from paper_2509_26581_b200 import _abi, bal

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")


@pytest.fixture(scope="module")
def ka():
    with open(os.path.join(GOLD, "known_answers.json")) as f:
        return json.load(f)


@pytest.fixture(scope="module")
def tiny():
    return dict(np.load(os.path.join(GOLD, "tiny_fp64.npz")))


def tiny_problem(t):
    return bal.BALProblem(t["cameras"], t["points"], t["camera_index"], t["point_index"], t["observations"])


# ----------------------------------------------------------- C ABI surface
def test_abi_exports_every_declared_symbol():
    header = open(os.path.join(ROOT, "include", "gb_bal.h")).read()
    header += open(os.path.join(ROOT, "include", "gb_generic.h")).read()
    declared = set(re.findall(r"\b(gbg?_[a-z_0-9]+)\s*\(", header))
    assert declared == set(_abi.EXPORTED)
    lib = ctypes.CDLL(_abi.LIB_PATH)
    for name in declared:
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", _abi.LIB_PATH], capture_output=True, text=True).stdout
    for name in declared:
        assert re.search(rf"\bT {name}\b", out), name


def test_no_cpu_fallback_without_device():
    L = _abi.lib()
    if L.gb_device_count() > 0:
        pytest.skip("a GPU is visible")
    assert not L.gb_create(_abi.GB_FP64, _abi.GB_ANALYTIC, 0)
    assert b"no CPU fallback" in L.gb_last_error()
    with pytest.raises(bal.DeviceError):
        bal.build_graph(bal.synthetic_bal(4, 10, 30), "fp64")


def test_default_config_matches_reference_defaults():
    c = _abi.gb_lm_config()
    _abi.lib().gb_default_config(ctypes.byref(c))
    py = bal.LMConfig().to_c()
    for f, _ in _abi.gb_lm_config._fields_:
        if f == "pcg":
            for g, _ in _abi.gb_pcg_config._fields_:
                assert getattr(c.pcg, g) == getattr(py.pcg, g)
        else:
            assert getattr(c, f) == getattr(py, f), f
    assert (c.max_iterations, c.pcg.max_iterations, c.tau) == (10, 50, 1e-4)


# ------------------------------------------------------ known answers (oracle)
def test_snavely_closed_forms(ka):
    # tests/test_bal.cpp:120-137
    cam = [0, 0, 0, 0, 0, 0, 100.0, 0, 0]
    assert np.array_equal(R.project(cam, [0, 0, -1]), [0, 0]) and ka["project_origin"] == [0, 0]
    assert abs(R.project(cam, [1, 0, -1])[0] - 100.0) <= 1e-12 and abs(ka["project_x1"][0] - 100) <= 1e-12
    cam[7] = 0.1
    assert abs(R.project(cam, [1, 0, -1])[0] - 110.0) <= 1e-12 and abs(ka["project_k1"][0] - 110) <= 1e-12


def test_rodrigues_known_rotation(ka):
    # tests/test_bal.cpp:139-147
    y = R.rotate(np.array([[0, 0, np.pi / 2]]), np.array([[1.0, 0, 0]]), R.Prec("fp64"))[0]
    assert abs(y[0]) < 1e-14 and abs(y[1] - 1) < 1e-14 and abs(y[2]) < 1e-15
    assert np.allclose(y, ka["rotate_half_pi"], atol=1e-15)


def test_nielsen_schedule(ka):
    # tests/test_lm_optimizer.cpp:13-29
    got = [R.update_damping(1.0, 2.0, False, 0.0), R.update_damping(3.0, 4.0, True, 1.0),
           R.update_damping(3.0, 2.0, True, 0.5)]
    assert got == [tuple(x) for x in ka["nielsen"]] == [(2.0, 4.0), (1.0, 2.0), (3.0, 2.0)]


def test_bf16_rounding(ka):
    # bfloat16.hpp:25-33 (RNE, quiet NaN with sign)
    for v, bits in ka["bf16"]:
        assert int(R.bf16_round(np.float32(v)).view(np.uint32) >> 16) == bits
    assert int(R.bf16_round(np.float32("nan")).view(np.uint32) >> 16) == ka["bf16_nan"] == 0x7FC0


def test_jacobians_known_and_finite_difference(ka):
    # tests/test_bal.cpp:202-246: analytic vs FD < 1e-5; restatement vs reference
    P = R.Prec("fp64")
    for case in ka["jacobian_cases"]:
        c = np.array(case["camera"])[None]
        x = np.array(case["point"])[None]
        jc, jp = R.jacobians(c, x, P)
        assert np.linalg.norm(jc.reshape(-1) - case["jc"]) <= 1e-12 * np.linalg.norm(case["jc"])
        assert np.linalg.norm(jp.reshape(-1) - case["jp"]) <= 1e-12 * np.linalg.norm(case["jp"])
    rng = np.random.default_rng(44)
    checked = 0
    while checked < 200:
        c = np.concatenate([rng.normal(0, 0.4, 3), rng.normal(0, 1, 3), [rng.uniform(300, 1500)],
                            [rng.normal(0, 0.1)], [rng.normal(0, 0.01)]])
        x = rng.normal(0, 2, 3)
        if R.rotate(c[None, :3], x[None], P)[0, 2] + c[5] >= -0.1:
            continue
        checked += 1
        jc, jp = R.jacobians(c[None], x[None], P)
        fd = np.zeros((2, 12))
        z = np.concatenate([c, x])
        for k in range(12):
            h = max(1e-6, 1e-6 * abs(z[k]))
            zp, zm = z.copy(), z.copy()
            zp[k] += h
            zm[k] -= h
            fd[:, k] = (R.project(zp[:9], zp[9:]) - R.project(zm[:9], zm[9:])) / (2 * h)
        an = np.concatenate([jc[0], jp[0]], 1)
        assert np.linalg.norm(an - fd) / np.linalg.norm(fd) < 1e-5


# ------------------------------------------------- golden fixtures (oracle)
def test_restatement_reproduces_golden_tiny(tiny):
    g = R.build_graph(tiny_problem(tiny), "fp64")
    R.activate(g, 0)
    for (vos, off, items), k in zip(g.inc, ("cam", "pt")):
        assert np.array_equal(vos, tiny[f"{k}_vos"]) and np.array_equal(off, tiny[f"{k}_off"])
        assert np.array_equal(items, tiny[f"{k}_items"])
    ls = R.LinearSystem(g)
    chi = ls.linearize()
    assert abs(chi - tiny["chi2"]) <= 1e-13 * tiny["chi2"]
    for k, v in (("b", ls.b), ("diag", ls.diag), ("scaling", ls.D)):
        assert np.linalg.norm(v - tiny[k]) <= 1e-12 * np.linalg.norm(tiny[k]), k
    jac = np.concatenate([ls.Jc.reshape(-1, 18), ls.Jp.reshape(-1, 6)], 1)
    assert np.linalg.norm(jac - tiny["jacobians"]) <= 1e-13 * np.linalg.norm(tiny["jacobians"])
    hv = ls.hvp(tiny["hvp_v"], 0.25)
    assert np.linalg.norm(hv - tiny["hvp_out"]) <= 1e-13 * np.linalg.norm(tiny["hvp_out"])
    blocks = ls.build_preconditioner(1e-3)
    assert np.linalg.norm(blocks - tiny["precond"]) <= 1e-9 * np.linalg.norm(tiny["precond"])
    dx, st, pred, fin = ls.solve_step(1e-3, dict(max_iterations=10, tolerance=1e-6, rejection_ratio=10,
                                                 normalize_rhs=True))
    assert st["iterations"] == int(tiny["pcg_its"])
    assert np.linalg.norm(dx - tiny["dx"]) <= 1e-9 * np.linalg.norm(tiny["dx"])
    g2 = R.build_graph(tiny_problem(tiny), "fp64")
    rep = R.levenberg_marquardt(g2, R.lm_config(50, 10))
    tr = tiny["trace"]
    assert len(rep["iterations"]) == tr.shape[0] and rep["termination"] == str(tiny["termination"])
    for it, row in zip(rep["iterations"], tr):
        assert abs(it["chi2_after"] - row[1]) <= 1e-10 * abs(row[1])
        assert it["pcg_iterations"] == int(row[3]) and it["accepted"] == bool(row[4])
    assert np.linalg.norm(g2.cams - tiny["final_cameras"]) <= 1e-10 * np.linalg.norm(tiny["final_cameras"])


def test_ref_reproduces_golden_tiny(ref, tiny):
    r = ref.build_graph(tiny_problem(tiny), "fp64")
    cfg = bal.LMConfig(max_iterations=50)
    cfg.pcg.max_iterations = 10
    rep = bal.levenberg_marquardt(r, cfg)
    assert rep.final_chi2 == float(tiny["final_chi2"])
    assert np.array_equal(r.cameras, tiny["final_cameras"])


@pytest.mark.parametrize("precision", ["fp64", "fp32", "fp32-bf16"])
def test_restatement_linear_system_vs_reference(ref, precision):
    p = bal.synthetic_bal(10, 120, 600, seed=5)
    r = ref.build_graph(p, precision)
    lr = r.ls_linearize(0)
    g = R.build_graph(p, precision)
    R.activate(g, 0)
    ls = R.LinearSystem(g)
    chi = ls.linearize()
    tol = 1e-13 if precision == "fp64" else 1e-5
    assert abs(chi - lr["chi2"]) <= tol * lr["chi2"]
    btol = 1e-11 if precision == "fp64" else 1e-3
    assert np.linalg.norm(ls.b - lr["b"]) <= btol * np.linalg.norm(lr["b"])
    v = np.random.default_rng(2).standard_normal(lr["n"])
    vs = v if precision != "fp32-bf16" else (R.bf16_round(v.astype(np.float32)).view(np.uint32) >> 16).astype(np.uint16)
    href = r.ls_hvp(vs, 0.1)
    vin = v.astype(ls.g.P.FP) if precision != "fp32-bf16" else R.bf16_round(v.astype(np.float32))
    hres = ls.hvp(vin, 0.1)
    assert np.linalg.norm(hres - href) <= btol * np.linalg.norm(href)


def test_restatement_lm_vs_reference_fp64(ref):
    for shape, seed in (((8, 60, 300), 11), ((20, 400, 2000), 3)):
        p = bal.synthetic_bal(*shape, seed=seed)
        rep_r = bal.levenberg_marquardt(ref.build_graph(p, "fp64"), _bal_cfg())
        rep_s = R.levenberg_marquardt(R.build_graph(p, "fp64"), R.lm_config(50, 10))
        assert len(rep_s["iterations"]) == len(rep_r.iterations) and rep_s["termination"] == rep_r.termination
        assert abs(rep_s["final_chi2"] - rep_r.final_chi2) <= 1e-10 * rep_r.final_chi2


def _bal_cfg(its=50):
    c = bal.LMConfig(max_iterations=its)
    c.pcg.max_iterations = 10
    return c


def test_restatement_fixed_and_levels_vs_reference(ref):
    p = bal.synthetic_bal(12, 200, 1000, seed=8)
    rng = np.random.default_rng(1)
    cf, pf = np.zeros(12, bool), rng.random(200) < 0.1
    cf[0] = True
    lv = (rng.random(1000) < 0.1).astype(np.uint8)
    r = ref.build_graph(p, "fp64")
    r.set_fixed(cameras=cf, points=pf)
    r.set_levels(lv)
    rep_r = bal.levenberg_marquardt(r, _bal_cfg())
    g = R.build_graph(p, "fp64", cam_fixed=cf, pt_fixed=pf, levels=lv)
    rep_s = R.levenberg_marquardt(g, R.lm_config(50, 10))
    assert len(rep_s["iterations"]) == len(rep_r.iterations)
    assert abs(rep_s["final_chi2"] - rep_r.final_chi2) <= 1e-10 * rep_r.final_chi2
    r.ls_linearize(0)
    for which in (0, 1):
        a = r.incidence(which)
        b = g.inc[which]
        for x, y in zip(a[:3], b):
            assert np.array_equal(x, y)


# ----------------------------------------------------------------- host logic
def test_synthetic_generator_shape_and_determinism():
    for (nc, np_, ne) in ((49, 7776, 31843), (24, 600, 3600)):
        p = bal.synthetic_bal(nc, np_, ne, seed=42)
        q = bal.synthetic_bal(nc, np_, ne, seed=42)
        assert np.array_equal(p.observations, q.observations) and np.array_equal(p.cameras, q.cameras)
        assert p.num_observations == ne and p.num_points == np_ and p.num_cameras == nc
        deg = np.bincount(p.point_index, minlength=np_)
        base, extra = divmod(ne, np_)
        assert np.all(deg[:extra] == base + 1) and np.all(deg[extra:] == base)
        assert np.all(np.diff(p.point_index.astype(np.int64)) >= 0)  # point-grouped, as in BAL files
        for pt in range(0, np_, max(1, np_ // 50)):  # distinct cameras per point
            cams = p.camera_index[p.point_index == pt]
            assert len(set(cams.tolist())) == len(cams)
    assert not np.array_equal(bal.synthetic_bal(24, 600, 3600, seed=1).observations,
                              bal.synthetic_bal(24, 600, 3600, seed=2).observations)
    with pytest.raises(ValueError):
        bal.synthetic_bal(4, 10, 5)  # fewer observations than points


def test_synthetic_initial_estimate_is_a_perturbation(ref):
    p = bal.synthetic_bal(24, 600, 3600, seed=42)
    r = ref.build_graph(p, "fp64")
    mse0 = r.mse()
    rep = bal.levenberg_marquardt(r, _bal_cfg(30))
    assert 1.0 < mse0 < 1e4 and 0.5 < r.mse() < 2.5  # ~1 px noise per axis after convergence
    assert rep.accepted_steps >= 3


def test_zipf_variant_skews_camera_degrees():
    p = bal.synthetic_bal(200, 5000, 25000, seed=4, zipf=1.1)
    deg = np.bincount(p.camera_index, minlength=200)
    assert deg.max() > 5 * np.median(deg)


def test_bal_text_round_trip():
    p = bal.synthetic_bal(5, 40, 160, seed=9)
    q = bal.parse_bal_text(bal.serialize_bal_text(p))
    for a, b in ((p.cameras, q.cameras), (p.points, q.points), (p.observations, q.observations)):
        assert np.array_equal(a, b)
    assert np.array_equal(p.camera_index, q.camera_index)
    with pytest.raises(ValueError):
        bal.parse_bal_text("2 2 1\n0 5 1.0 2.0\n" + "0\n" * 24)


def test_reference_memory_account_ratios(ref):
    # tests/test_bench.cpp:63-88 / SPEC acceptance 5
    p = bal.synthetic_bal(10, 100, 500, seed=1)
    acc = {}
    for prec, mode in (("fp32", "analytic"), ("fp32-bf16", "analytic"), ("fp64", "dynamic")):
        acc[(prec, mode)] = bal.levenberg_marquardt(ref.build_graph(p, prec, mode), _bal_cfg(1)).memory
    assert acc[("fp32", "analytic")]["jacobian_bytes"] == 500 * 24 * 4
    assert acc[("fp32-bf16", "analytic")]["jacobian_bytes"] * 2 == acc[("fp32", "analytic")]["jacobian_bytes"]
    assert acc[("fp64", "dynamic")]["jacobian_bytes"] == 0


# --------------------------------------------- Schur mode (its own oracle)
def test_schur_restatement_against_dense():
    p = bal.synthetic_bal(6, 40, 200, seed=12)
    g = R.build_graph(p, "fp64")
    R.activate(g, 0)
    ls = R.LinearSystem(g)
    ls.linearize()
    sch = R.SchurSystem(ls)
    lam = 0.05
    A, S, r, xdense, rhs = sch.dense(lam)
    Sop = sch.operator(lam)
    nc9 = 9 * sch.nfc
    E = np.eye(nc9)
    Smf = np.stack([Sop(E[k]) for k in range(nc9)], 1)
    assert np.linalg.norm(Smf - S) <= 1e-10 * np.linalg.norm(S)
    # converged Schur PCG == dense solve of the full damped system
    pcg = dict(max_iterations=200, tolerance=1e-13, rejection_ratio=10, normalize_rhs=True)
    dx, st, pred, fin = sch.solve_step(lam, pcg)
    x = np.linalg.solve(A, rhs)
    assert np.allclose(xdense, x, rtol=1e-9, atol=1e-12)
    assert np.linalg.norm(dx - ls.D * x) <= 1e-8 * np.linalg.norm(ls.D * x)
    assert st["converged"]
