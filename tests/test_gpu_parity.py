"""Parity of the B200 path against the compiled reference (oracle/_ref).

Every test here runs the device solver through the C ABI and the unmodified
reference solver on the same synthetic BAL problem, and compares the
quantities the reference's own suites pin (tests/test_linear_system.cpp,
tests/test_lm_optimizer.cpp, tests/acceptance.cpp) at the tolerances
BASELINE.json's north star states: index structures bit-exact; final chi^2
within 1e-6 relative (fp64) / 1e-4 (fp32, fp32-bf16) with the same LM
iteration count.
"""
import ctypes

import numpy as np
import pytest

from paper_2509_26581_b200 import bal

pytestmark = pytest.mark.gpu

LADYBUG = (49, 7776, 31843)
TINY = (8, 60, 300)


def rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def bal_cfg(max_it=50, pcg_it=10):
    c = bal.LMConfig(max_iterations=max_it)
    c.pcg.max_iterations = pcg_it
    c.pcg.tolerance = 1e-6
    return c


@pytest.fixture(scope="module")
def ladybug():
    return bal.synthetic_bal(*LADYBUG, seed=42)


def pair(problem, ref, precision="fp64", mode="analytic", huber=None, fixed=None, levels=None):
    g = bal.build_graph(problem, precision, mode, huber)
    r = ref.build_graph(problem, precision, mode, huber, workers=4)
    for x in (g, r):
        if fixed is not None:
            x.set_fixed(cameras=fixed[0], points=fixed[1])
        if levels is not None:
            x.set_levels(levels)
    return g, r


def test_incidence_bit_exact(gpu, ref, ladybug):
    rng = np.random.default_rng(5)
    fixed = (rng.random(LADYBUG[0]) < 0.1, rng.random(LADYBUG[1]) < 0.05)
    levels = (rng.random(LADYBUG[2]) < 0.03).astype(np.uint8)
    for fx, lv in ((None, None), (fixed, levels)):
        g, r = pair(ladybug, ref, fixed=fx, levels=lv)
        g.ls_linearize(0)
        r.ls_linearize(0)
        for which in (0, 1):
            a, b = g.incidence(which), r.incidence(which)
            for x, y in zip(a, b):
                assert x.dtype == y.dtype and np.array_equal(x, y)


@pytest.mark.parametrize("precision", ["fp64", "fp32", "fp32-bf16"])
def test_linearize_parity(gpu, ref, ladybug, precision):
    g, r = pair(ladybug, ref, precision)
    a, b = g.ls_linearize(0), r.ls_linearize(0)
    tol = 1e-12 if precision == "fp64" else 2e-5
    assert a["n"] == b["n"] and a["finite"] == b["finite"]
    assert abs(a["chi2"] - b["chi2"]) <= tol * abs(b["chi2"])
    # b/diag tolerances: accumulated at FP, association order differs
    gtol = 1e-10 if precision == "fp64" else (2e-4 if precision == "fp32" else 2e-2)
    for k in ("b", "diag", "clamped", "scaling"):
        assert rel(a[k], b[k]) <= gtol, k


def test_jacobians_parity(gpu, ref, ladybug):
    g, r = pair(ladybug, ref)
    g.ls_linearize(0)
    r.ls_linearize(0)
    ja, jb = g.ls_jacobians(LADYBUG[2]), r.ls_jacobians(LADYBUG[2])
    assert rel(ja, jb) <= 1e-12


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_factored_jacobian_store_bit_exact(gpu, ladybug, monkeypatch, precision):
    """The factored J store (16 values per edge + R, f per camera; DESIGN.md
    §2) rebuilds exactly the chain's J: bit-identical to the full 24-value
    store, and the HVP / LM trace through it is bit-identical too."""
    out = {}
    monkeypatch.setenv("GB_HVP_RC", "0")  # the stored-J path
    for jf in ("1", "0"):
        monkeypatch.setenv("GB_JFACT", jf)
        g = bal.build_graph(ladybug, precision, "analytic")
        n = g.ls_linearize(0)["n"]
        v = np.random.default_rng(3).standard_normal(n)
        out[jf] = (g.ls_jacobians(LADYBUG[2]), g.ls_hvp(v, 1e-3))
        g2 = bal.build_graph(ladybug, precision, "analytic")
        rep = bal.levenberg_marquardt(g2, bal_cfg(8))
        out[jf] += ([(i.chi2_after, i.lambda_, i.pcg_iterations) for i in rep.iterations], g2.cameras.copy())
    a, b = out["1"], out["0"]
    assert np.array_equal(a[0].view(np.uint8), b[0].view(np.uint8))
    assert np.array_equal(a[1], b[1])
    assert a[2] == b[2]
    assert np.array_equal(a[3], b[3])


@pytest.mark.parametrize("precision,mode,huber", [("fp64", "analytic", None), ("fp64", "auto", None),
                                                 ("fp32", "analytic", 2.0), ("fp32-bf16", "analytic", None)])
def test_pipelined_hvp_bit_exact(gpu, monkeypatch, precision, mode, huber):
    """The bulk-copy pipelined HVP (hvp_pipe.cuh) keeps k_hvp_tiles' arithmetic
    and association order: bit-identical HVP and LM trace with it on and off.
    Problem sized to give several tiles per CTA (ring wrap-around) and heavy
    tiles (a point seen by > 512 cameras)."""
    probs = [bal.synthetic_bal(900, 60000, 330000, seed=11), bal.synthetic_bal(900, 60000, 330000, seed=12, zipf=1.2)]
    for p in probs:
        _pipe_vs_tiles(monkeypatch, p, precision, mode, huber)


def _pipe_vs_tiles(monkeypatch, p, precision, mode, huber):
    out = {}
    monkeypatch.setenv("GB_HVP_RC", "0")  # the stored-J path
    for pipe in ("1", "0"):
        monkeypatch.setenv("GB_HVP_PIPE", pipe)
        g = bal.build_graph(p, precision, mode, huber)
        n = g.ls_linearize(0)["n"]
        v = np.random.default_rng(4).standard_normal(n)
        h = g.ls_hvp(v, 1e-3)
        g2 = bal.build_graph(p, precision, mode, huber)
        rep = bal.levenberg_marquardt(g2, bal_cfg(4))
        out[pipe] = (h, [(i.chi2_after, i.lambda_, i.pcg_iterations) for i in rep.iterations], g2.points.copy())
    assert np.array_equal(out["1"][0], out["0"][0])
    assert out["1"][1] == out["0"][1]
    assert np.array_equal(out["1"][2], out["0"][2])


@pytest.mark.parametrize("precision,mode,huber,zipf", [("fp64", "analytic", None, None), ("fp64", "analytic", 2.0, 1.2),
                                                      ("fp64", "dynamic", None, None), ("fp32", "analytic", 2.0, None),
                                                      ("fp32-bf16", "dynamic", None, None)])
def test_recompute_hvp(gpu, monkeypatch, precision, mode, huber, zipf):
    """The recompute HVP (hvp_rc.cuh: no Jacobian store, the factored
    operator applied per camera run) against the stored-J pipeline: the same
    operator to rounding, the same LM trace (iterations, accept pattern, PCG
    iterations) and final cost. Several tiles per CTA, heavy tiles (a point
    seen by > 512 cameras) and skewed camera degrees."""
    p = bal.synthetic_bal(900, 60000, 330000, seed=11, zipf=zipf) if zipf else bal.synthetic_bal(900, 60000, 330000, seed=11)
    out = {}
    for rc in ("1", "0"):
        monkeypatch.setenv("GB_HVP_RC", rc)
        g = bal.build_graph(p, precision, mode, huber)
        n = g.ls_linearize(0)["n"]
        path = ctypes.c_int32()
        g.backend.check(g.backend.fn("hvp_info")(g._h, ctypes.byref(path), None, None, None))
        assert path.value == (3 if rc == "1" else (0 if mode == "dynamic" else 2)), path.value  # the path under test
        v = np.random.default_rng(4).standard_normal(n)
        hs = [g.ls_hvp(v, lam) for lam in (0.0, 1e-3)]
        g2 = bal.build_graph(p, precision, mode, huber)
        rep = bal.levenberg_marquardt(g2, bal_cfg(6))
        out[rc] = (hs, rep, g2.points.copy(), g2.cameras.copy())
    # bf16 storage: the HVP output is narrowed to bf16, so float-rounding differences
    # of the two association orders can move an entry by one bf16 ulp (2^-8)
    tol = {"fp64": 1e-12, "fp32": 2e-5, "fp32-bf16": 1e-2}[precision]
    for a, b in zip(out["1"][0], out["0"][0]):
        assert rel(a, b) <= tol
    ra, rb = out["1"][1], out["0"][1]
    assert ra.termination == rb.termination and len(ra.iterations) == len(rb.iterations)
    assert [i.accepted for i in ra.iterations] == [i.accepted for i in rb.iterations]
    if precision != "fp32-bf16":
        assert [i.pcg_iterations for i in ra.iterations] == [i.pcg_iterations for i in rb.iterations]
    ctol = {"fp64": 1e-9, "fp32": 1e-4, "fp32-bf16": 1e-3}[precision]
    assert abs(ra.final_chi2 - rb.final_chi2) <= ctol * rb.final_chi2
    assert rel(out["1"][2], out["0"][2]) <= {"fp64": 1e-7, "fp32": 1e-3, "fp32-bf16": 1e-2}[precision]


@pytest.mark.parametrize("precision,huber", [("fp64", None), ("fp32", 2.0)])
def test_deferred_x_update_bit_exact(gpu, monkeypatch, precision, huber):
    """PCG's x += alpha p deferred into the next HVP (defer_x) evaluates the
    same expression on the same operands as the in-place update: the LM trace
    and the refined parameters are bit-identical with it on and off."""
    p = bal.synthetic_bal(900, 60000, 330000, seed=11)
    out = {}
    for dx in ("1", "0"):
        monkeypatch.setenv("GB_DEFER_X", dx)
        g = bal.build_graph(p, precision, "analytic", huber)
        rep = bal.levenberg_marquardt(g, bal_cfg(5))
        out[dx] = ([(i.chi2_after, i.lambda_, i.pcg_iterations) for i in rep.iterations], g.points.copy(),
                   g.cameras.copy())
    assert out["1"][0] == out["0"][0]
    assert np.array_equal(out["1"][1], out["0"][1]) and np.array_equal(out["1"][2], out["0"][2])


def test_recompute_hvp_deterministic(gpu, monkeypatch):
    """Fixed association order everywhere: two runs are bit-identical."""
    monkeypatch.setenv("GB_HVP_RC", "1")
    p = bal.synthetic_bal(300, 20000, 110000, seed=5)
    res = []
    for _ in range(2):
        g = bal.build_graph(p, "fp64", "analytic")
        n = g.ls_linearize(0)["n"]
        res.append(g.ls_hvp(np.random.default_rng(2).standard_normal(n), 1e-3))
    assert np.array_equal(res[0], res[1])


@pytest.mark.parametrize("mode", ["analytic", "dynamic"])
def test_hvp_parity(gpu, ref, ladybug, mode):
    g, r = pair(ladybug, ref, mode=mode)
    n = g.ls_linearize(0)["n"]
    r.ls_linearize(0)
    rng = np.random.default_rng(1)
    for lam in (0.0, 1e-4, 0.37):
        v = rng.standard_normal(n)
        assert rel(g.ls_hvp(v, lam), r.ls_hvp(v, lam)) <= 1e-12


def test_preconditioner_parity(gpu, ref, ladybug):
    g, r = pair(ladybug, ref)
    g.ls_linearize(0)
    r.ls_linearize(0)
    for lam in (1e-4, 0.05):
        ba, fa = g.ls_preconditioner(lam, LADYBUG[0], LADYBUG[1])
        bb, fb = r.ls_preconditioner(lam, LADYBUG[0], LADYBUG[1])
        assert fa == fb
        assert rel(ba, bb) <= 1e-9


def test_solve_step_parity(gpu, ref, ladybug):
    g, r = pair(ladybug, ref)
    g.ls_linearize(0)
    r.ls_linearize(0)
    for lam, its in ((1e-4, 10), (1e-2, 50)):
        pcg = bal.PCGConfig(max_iterations=its)
        dxa, sa, pa, fa = g.ls_solve_step(lam, pcg)
        dxb, sb, pb, fb = r.ls_solve_step(lam, pcg)
        assert sa["iterations"] == sb["iterations"] and sa["converged"] == sb["converged"] and fa == fb
        assert rel(dxa, dxb) <= 1e-8
        assert abs(pa - pb) <= 1e-8 * abs(pb)


def run_pair(problem, ref, precision="fp64", mode="analytic", cfg=None, **kw):
    cfg = cfg or bal_cfg()
    g, r = pair(problem, ref, precision, mode, **kw)
    ra = bal.levenberg_marquardt(g, cfg)
    rb = bal.levenberg_marquardt(r, cfg)
    return g, r, ra, rb


def assert_trace_parity(ra, rb, tol):
    assert ra.termination == rb.termination
    assert len(ra.iterations) == len(rb.iterations)
    assert [i.accepted for i in ra.iterations] == [i.accepted for i in rb.iterations]
    assert abs(ra.initial_chi2 - rb.initial_chi2) <= tol * rb.initial_chi2
    assert abs(ra.final_chi2 - rb.final_chi2) <= tol * rb.final_chi2
    for x, y in zip(ra.iterations, rb.iterations):
        if np.isfinite(y.chi2_after):
            assert abs(x.chi2_after - y.chi2_after) <= tol * abs(y.chi2_after)
    assert ra.accepted_steps == rb.accepted_steps


def test_lm_parity_fp64(gpu, ref, ladybug):
    g, r, ra, rb = run_pair(ladybug, ref)
    assert_trace_parity(ra, rb, 1e-6)
    for x, y in zip(ra.iterations, rb.iterations):
        assert x.pcg_iterations == y.pcg_iterations
        assert abs(x.lambda_ - y.lambda_) <= 1e-6 * y.lambda_
    assert rel(g.cameras, r.cameras) <= 1e-6 and rel(g.points, r.points) <= 1e-6
    assert abs(g.mse() - r.mse()) <= 1e-6 * r.mse()
    assert ra.memory == rb.memory
    assert ra.free_dims == rb.free_dims and ra.active_factors == rb.active_factors


@pytest.mark.parametrize("precision", ["fp32", "fp32-bf16"])
def test_lm_parity_low_precision(gpu, ref, ladybug, precision):
    # At tolerance 1e-4 (resolvable in float) the LM trace is decided by the
    # algorithm: same iteration count and accept pattern as the reference.
    cfg = bal_cfg()
    cfg.tolerance = 1e-4
    g, r, ra, rb = run_pair(ladybug, ref, precision, cfg=cfg)
    assert ra.termination == rb.termination
    assert len(ra.iterations) == len(rb.iterations)
    assert [i.accepted for i in ra.iterations] == [i.accepted for i in rb.iterations]
    assert abs(ra.final_chi2 - rb.final_chi2) <= 1e-4 * rb.final_chi2
    assert ra.memory == rb.memory
    # At the BAL config's 1e-6 the reference's own float chi^2 (a sequential
    # sum) carries ~3e-6 relative rounding noise, so the last accept/terminate
    # decision is noise-decided (a faithful numpy restatement also differs by
    # one iteration, tests/test_oracle_cpu.py); cost parity still holds.
    g, r, ra, rb = run_pair(ladybug, ref, precision)
    assert abs(ra.final_chi2 - rb.final_chi2) <= 1e-4 * rb.final_chi2


def test_lm_parity_dynamic(gpu, ref, ladybug):
    g, r, ra, rb = run_pair(ladybug, ref, mode="dynamic")
    assert_trace_parity(ra, rb, 1e-6)
    assert ra.memory["jacobian_bytes"] == 0 == rb.memory["jacobian_bytes"]


def test_lm_parity_huber(gpu, ref, ladybug):
    g, r, ra, rb = run_pair(ladybug, ref, huber=2.0)
    assert_trace_parity(ra, rb, 1e-6)


def test_fixed_vertices_and_levels(gpu, ref, ladybug):
    rng = np.random.default_rng(9)
    fixed = (np.zeros(LADYBUG[0], bool), rng.random(LADYBUG[1]) < 0.05)
    fixed[0][:3] = True
    levels = (rng.random(LADYBUG[2]) < 0.05).astype(np.uint8)
    cams0 = ladybug.cameras.copy()
    pts0 = ladybug.points.copy()
    g, r, ra, rb = run_pair(ladybug, ref, fixed=fixed, levels=levels)
    assert_trace_parity(ra, rb, 1e-6)
    # fixed vertices bit-identical end to end (tests/test_lm_optimizer.cpp:203-210)
    assert np.array_equal(g.cameras[fixed[0]].view(np.uint64), cams0[fixed[0]].view(np.uint64))
    assert np.array_equal(g.points[fixed[1]].view(np.uint64), pts0[fixed[1]].view(np.uint64))


def test_deterministic(gpu, ladybug):
    outs = []
    for _ in range(2):
        g = bal.build_graph(ladybug, "fp64")
        rep = bal.levenberg_marquardt(g, bal_cfg(8))
        outs.append((g.cameras.copy(), g.points.copy(), [i.chi2_after for i in rep.iterations]))
    assert np.array_equal(outs[0][0].view(np.uint64), outs[1][0].view(np.uint64))
    assert np.array_equal(outs[0][1].view(np.uint64), outs[1][1].view(np.uint64))
    assert outs[0][2] == outs[1][2]


def test_page_locked_graph_arrays(gpu, ladybug):
    """bal::BalGraph's own arrays (adapter.hpp:82-90) live in gb_host_alloc
    memory; an array kept past its graph stays valid (the block is not handed
    to the next graph while any view of it is alive)."""
    g = bal.build_graph(ladybug, "fp64")
    owner = g.cameras
    while owner is not None and not isinstance(owner, bal._PinnedBlock):
        owner = getattr(owner, "base", None)
    assert owner is not None and owner.ptr
    bal.levenberg_marquardt(g, bal_cfg(3))
    kept = g.cameras
    snap = kept.copy()
    del g
    g2 = bal.build_graph(ladybug, "fp64")
    bal.levenberg_marquardt(g2, bal_cfg(5))
    assert np.array_equal(kept.view(np.uint64), snap.view(np.uint64))
    assert not np.shares_memory(kept, g2.cameras)


def test_non_finite_initial_chi2_raises(gpu):
    p = bal.synthetic_bal(*TINY, seed=3)
    p.points[0] = [0.0, 0.0, 0.0]
    p.cameras[p.camera_index[0]][3:6] = 0.0  # P_z = 0 for the first observation -> inf
    g = bal.build_graph(p, "fp64")
    with pytest.raises(RuntimeError, match="non-finite chi\\^2"):
        bal.levenberg_marquardt(g, bal_cfg(3))


def test_tiny_and_heavy_tiles(gpu, ref):
    # points with > kTileEdges observations take the heavy-tile path
    p = bal.synthetic_bal(520, 30, 30 * 520, seed=7)
    for prob in (bal.synthetic_bal(*TINY, seed=11), p):
        g, r, ra, rb = run_pair(prob, ref, cfg=bal_cfg(12))
        assert_trace_parity(ra, rb, 1e-6)


def test_stepping_api_matches_optimize(gpu, ladybug):
    import ctypes

    from paper_2509_26581_b200 import _abi

    cfg = bal_cfg(8)
    g1 = bal.build_graph(ladybug, "fp64")
    r1 = bal.levenberg_marquardt(g1, cfg)
    g2 = bal.build_graph(ladybug, "fp64")
    L = g2.backend
    c = cfg.to_c()
    L.check(L.fn("begin")(g2._h, ctypes.byref(c), None))
    for _ in range(8):
        L.check(L.fn("step")(g2._h, 1))
    rep = _abi.gb_solve_report()
    L.check(L.fn("end")(g2._h, ctypes.byref(rep), None, 0))
    assert rep.final_chi2 == r1.final_chi2 and rep.iterations_run == len(r1.iterations)
    assert np.array_equal(g1.points, g2.points)
    ms = ctypes.c_double()
    L.check(L.fn("time_hvp")(g2._h, 3, ctypes.byref(ms), None))
    assert ms.value > 0


def test_device_activation_matches_host(gpu):
    from paper_2509_26581_b200 import _abi

    rng = np.random.default_rng(3)
    cases = [bal.synthetic_bal(*LADYBUG, seed=42), bal.synthetic_bal(520, 30, 30 * 520, seed=7),
             bal.synthetic_bal(*TINY, seed=5), bal.synthetic_bal(200, 5000, 25000, seed=4, zipf=1.1)]
    for i, p in enumerate(cases):
        g = bal.build_graph(p, "fp64")
        if i == 0:
            g.set_fixed(cameras=rng.random(p.num_cameras) < 0.1, points=rng.random(p.num_points) < 0.05)
            g.set_levels((rng.random(p.num_observations) < 0.05).astype(np.uint8))
        g.backend.check(_abi.lib().gb_activation_selfcheck(g._h, 0))


def test_auto_mode_parity(gpu, ref, ladybug):
    # DifferentiationMode::Auto: dual-number Jacobians (factor_descriptor.hpp:610-624);
    # analytic vs auto < 1e-12 (tests/test_bal.cpp:243-244), traces vs the reference's auto run
    ga, ra = pair(ladybug, ref, mode="auto")
    ga.ls_linearize(0)
    ra.ls_linearize(0)
    ja, jr = ga.ls_jacobians(LADYBUG[2]), ra.ls_jacobians(LADYBUG[2])
    assert rel(ja, jr) <= 1e-13
    gn, _ = pair(ladybug, ref)
    gn.ls_linearize(0)
    assert rel(ja, gn.ls_jacobians(LADYBUG[2])) <= 1e-12
    g, r, a1, b1 = run_pair(ladybug, ref, mode="auto")
    assert_trace_parity(a1, b1, 1e-6)


def test_large_problem_trace_parity(gpu, ref):
    # > 1 M columns: every vertex-, column- and tile-grid covers the whole
    # problem (small cases fit in one grid wave and would hide coverage bugs)
    p = bal.synthetic_bal(60, 400_000, 2_000_000, seed=8)
    cfg = bal_cfg(3)
    g = bal.build_graph(p, "fp64")
    ra = bal.levenberg_marquardt(g, cfg)
    r = ref.build_graph(p, "fp64", workers=16)
    rb = bal.levenberg_marquardt(r, cfg)
    assert [i.pcg_iterations for i in ra.iterations] == [i.pcg_iterations for i in rb.iterations]
    assert_trace_parity(ra, rb, 1e-6)


@pytest.mark.parametrize("variant", ["before_scaling", "no_guard", "refresh_on_reject", "no_normalize",
                                     "clamps", "tau_lambda_max", "loose_pcg"])
def test_lm_config_variants(gpu, ref, ladybug, variant):
    """Every LMConfig / PCGConfig / LinearSystemOptions field the reference
    exposes (levenberg_marquardt.hpp:15-26, pcg.hpp:12-17,
    linear_system.hpp:15-19) runs on the device with the reference's semantics:
    the same LM trace as the compiled reference."""
    cfg = bal_cfg(25)
    if variant == "before_scaling":
        cfg.damping = "before_scaling"
    elif variant == "no_guard":
        cfg.use_rejection_guard = False
        cfg.pcg.max_iterations = 3
    elif variant == "refresh_on_reject":
        cfg.refresh_on_reject = True
        cfg.tau = 1e-9  # tiny initial damping: early rejects
    elif variant == "no_normalize":
        cfg.pcg.normalize_rhs = False
    elif variant == "clamps":
        cfg.clamp_min, cfg.clamp_max = 1e-2, 1e6
    elif variant == "tau_lambda_max":
        cfg.tau, cfg.lambda_max = 10.0, 1e4
    elif variant == "loose_pcg":
        cfg.pcg.tolerance, cfg.pcg.rejection_ratio = 1e-2, 2.0
    g, r, ra, rb = run_pair(ladybug, ref, cfg=cfg)
    assert_trace_parity(ra, rb, 1e-6)
    assert [i.pcg_iterations for i in ra.iterations] == [i.pcg_iterations for i in rb.iterations]
    assert [i.low_quality_step for i in ra.iterations] == [i.low_quality_step for i in rb.iterations]


def _exact_problem(problem):
    """The problem's observations replaced by exact projections of its own
    initial parameters (zero residual start, test_lm_optimizer.cpp:115-126)."""
    from oracle import restatement as R

    q = problem.copy()
    cams = q.cameras[q.camera_index]
    pts = q.points[q.point_index]
    # binary64 Snavely predictions (snavely.hpp:48-61): residual against obs = 0
    q.observations[:] = R.residual(cams, pts, np.zeros((len(cams), 2)), R.Prec("fp64"))
    return q


@pytest.mark.parametrize("case", ["gradient_small", "damping_overflow", "no_free_parameters", "max_iterations"])
def test_terminations(gpu, ref, case):
    """Every Termination the reference's loop can report (levenberg_marquardt.hpp:28-35)
    is reached on the device with the reference's trace."""
    p = bal.synthetic_bal(*TINY, seed=21)
    cfg = bal_cfg(30)
    fixed = None
    if case == "gradient_small":
        # zero-residual start; the tolerance sits above the last-ulp residuals
        # (device sincos / FMA vs libm) that an exactly-zero threshold would see
        p = _exact_problem(p)
        cfg.gradient_tolerance = 1e-6
    elif case == "damping_overflow":
        cfg.lambda_max, cfg.tau = 1e-3, 1.0  # the first reject already overflows
        cfg.max_iterations = 30
    elif case == "no_free_parameters":
        fixed = (np.ones(TINY[0], bool), np.ones(TINY[1], bool))
    else:
        cfg.max_iterations, cfg.tolerance = 3, 0.0
    g, r = pair(p, ref, fixed=fixed)
    ra, rb = bal.levenberg_marquardt(g, cfg), bal.levenberg_marquardt(r, cfg)
    assert ra.termination == rb.termination
    if case != "damping_overflow":
        assert ra.termination == case
    if case == "gradient_small":  # chi^2 ~0: last-ulp residuals, compare absolutely
        assert len(ra.iterations) == len(rb.iterations) == 1
        assert ra.final_chi2 < 1e-18 and rb.final_chi2 < 1e-18
    else:
        assert_trace_parity(ra, rb, 1e-6)
