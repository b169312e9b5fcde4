"""Report wire format: gb_report_json / gb_report_csv against
the reference's own include/gopt/report.hpp (to_json(...).dump() with
nlohmann/json 3.11.3, and to_csv), compiled into oracle/_ref. Byte-equal on
a real reference solve report and on adversarial numbers (integral values,
the plain/scientific switch points, subnormals, signed zero, NaN / inf)."""
import ctypes
import json

import numpy as np
import pytest

from paper_2509_26581_b200 import _abi, bal


def wire(lib, prefix, kind, rep, recs, n):
    fn = getattr(lib, f"{prefix}report_{kind}")
    fn.restype = ctypes.c_int
    fn.argtypes = [ctypes.POINTER(_abi.gb_solve_report), ctypes.c_void_p, ctypes.c_int32, ctypes.c_char_p,
                   ctypes.c_uint64, ctypes.POINTER(ctypes.c_uint64)]
    need = ctypes.c_uint64()
    assert fn(ctypes.byref(rep), ctypes.cast(recs, ctypes.c_void_p), n, None, 0, ctypes.byref(need)) == 0
    buf = ctypes.create_string_buffer(need.value)
    assert fn(ctypes.byref(rep), ctypes.cast(recs, ctypes.c_void_p), n, buf, need.value, None) == 0
    return buf.value.decode()


@pytest.fixture(scope="module")
def reflib(ref):
    L = ref.lib()
    if not hasattr(L, "ref_report_json"):
        pytest.skip("oracle built without nlohmann/json")
    return L


def check(reflib, rep, recs, n):
    for kind in ("json", "csv"):
        a = wire(_abi.lib(), "gb_", kind, rep, recs, n)
        b = wire(reflib, "ref_", kind, rep, recs, n)
        assert a == b, (kind, a[:400], b[:400])


def test_report_of_a_reference_solve(ref, reflib):
    p = bal.synthetic_bal(12, 300, 1500, seed=42)
    c = bal.LMConfig(max_iterations=8)
    c.pcg.max_iterations = 10
    r = bal.levenberg_marquardt(ref.build_graph(p, "fp64", workers=2), c)
    rep, recs = r.to_c()
    check(reflib, rep, recs, len(r.iterations))
    d = json.loads(r.to_json())
    assert d["summary"]["iterations_run"] == len(r.iterations) and d["summary"]["termination"] == r.termination
    assert [it["lambda"] for it in d["iterations"]] == [it.lambda_ for it in r.iterations]
    assert r.to_csv().splitlines()[2].startswith("iteration,chi2_before,chi2_after,lambda,")


SPECIAL = [0.0, -0.0, 1.0, -1.0, 0.1, 1e-4, 1.5e-4, 1e-5, 9.99e-5, 123.456, 1e15, 1e16, 999999999999999.0,
           1234567890123456.0, 1e-300, 5e-324, 2.2250738585072014e-308, 1.7976931348623157e308, 1e300, 1e22,
           1e21, 0.30000000000000004, 2.0 / 3.0, 44480871.702812, 1e-7, float("nan"), float("inf"), -float("inf")]


def test_report_number_formats(reflib):
    rng = np.random.default_rng(1)
    vals = SPECIAL + list(rng.standard_normal(300) * 10.0 ** rng.integers(-30, 30, 300)) + \
        list(np.floor(rng.random(50) * 1e6))
    n = len(vals)
    recs = (_abi.gb_iteration_record * n)()
    for i, v in enumerate(vals):
        r = recs[i]
        r.iteration = i + 1
        r.chi2_before, r.chi2_after, r.lambda_ = v, -v, v * 3
        r.pcg_iterations, r.pcg_converged = i % 11, i % 2
        r.pcg_relative_residual = abs(v)
        r.low_quality_step, r.precond_fallback_blocks, r.accepted = i % 3 == 0, i % 5, i % 2
        r.wall_seconds = abs(v) if np.isfinite(v) else 0.0
    rep = _abi.gb_solve_report()
    rep.initial_chi2, rep.final_chi2 = 3590588700.377165, 44480871.70281
    rep.accepted_steps, rep.termination, rep.total_seconds = 21, 1, 0.375
    rep.free_dims, rep.residual_dims, rep.active_factors = 13491489, 57975288, 28987644
    rep.memory.jacobian_bytes, rep.memory.graph_bytes = 5565627648, 123
    for t in range(6):
        rep.termination = t
        check(reflib, rep, recs, n)
    check(reflib, rep, recs, 0)


def test_pow10_table_matches_nlohmann_header():
    """The Grisu2 cached powers (tools/gen_pow10.py) equal nlohmann's table."""
    import os
    import re

    h = "/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann/json.hpp"
    if not os.path.exists(h):
        pytest.skip("nlohmann header not present")
    theirs = [(int(f, 16), int(e), int(k)) for f, e, k in re.findall(r"\{0x([0-9A-F]+), (-?\d+), (-?\d+)\}",
                                                                      open(h).read())]
    from tools.gen_pow10 import table

    assert table() == theirs
