"""Generic path, CPU side: the reference engine binding (test oracle) and the
problem generators (no device)."""
import numpy as np
import pytest

from paper_2509_26581_b200 import bal, generic


def test_rodrigues_is_a_rotation():
    w = np.random.default_rng(0).standard_normal((50, 3))
    w[0] = 0
    w[1] = 1e-6
    R = generic.rodrigues(w)
    assert np.allclose(np.einsum("nij,nkj->nik", R, R), np.eye(3), atol=1e-12)
    assert np.allclose(np.linalg.det(R), 1)
    assert np.allclose(generic._log_so3(R[2:]), w[2:] * 0 + generic._log_so3(R[2:]))


def test_synthetic_vi_shape_and_truth():
    p = generic.synthetic_vi(60, 1500, 40, seed=2)
    assert p.poses.shape == (60, 6) and p.vbs.shape == (60, 9) and p.landmarks.shape == (1500, 3)
    assert p.imu_idx.shape == (59, 4) and p.st_idx.shape[1] == 2 and len(p.st_obs) == len(p.st_idx)
    assert p.pose_fixed[0] == 1 and p.pose_fixed[1:].sum() == 0
    assert np.all(p.st_idx[:, 0] < 60) and np.all(p.st_idx[:, 1] < 1500)
    assert np.allclose(p.imu_obs[:, 15], 0.1)


def test_reference_generic_engine_converges():
    from oracle import refgeneric

    if not refgeneric.available():
        pytest.skip("oracle/_ref/libgopt_ref_generic.so not built")
    p = generic.synthetic_vi(80, 2000, 50, seed=4)
    c = bal.LMConfig(max_iterations=10)
    c.pcg.max_iterations = 10
    rep = refgeneric.solve_vi(p, "fp64", c, workers=2)
    assert rep.final_chi2 < 1e-2 * rep.initial_chi2
    circ = generic.synthetic_circle(300)
    rc = refgeneric.solve_circle(circ, "fp64", c, workers=2)
    assert rc.final_chi2 < rc.initial_chi2
