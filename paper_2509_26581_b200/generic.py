"""Generic n-ary factor path: Python mirror of
include/gb_generic.h.

The reference's generic engine builds graphs from user vertex / factor traits
(vertex_descriptor.hpp:50-56, factor_descriptor.hpp:139-151) and solves them
with levenberg_marquardt (levenberg_marquardt.hpp:115-224). The device engine
(csrc/generic.cu) runs host-device traits (include/gb_generic_models.hpp) with
the same algorithm. Two models ship:

  circle  the reference toy (toy/circle.hpp:30-55), with its problem generator
  vi      an EuRoC-shaped global visual-inertial BA: stereo keyframes and IMU
          preintegration edges (BASELINE.json configs[4]); synthetic_vi()
          builds a problem of that shape (no dataset access here).
"""
import ctypes
from ctypes import POINTER, c_double, c_int, c_int32, c_uint64, c_void_p
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _abi
from .bal import LMConfig, SolveReport, _report

PREC = {"fp64": _abi.GB_FP64, "fp32": _abi.GB_FP32}


def _declare(lib, prefix):
    vp = c_void_p
    fn = getattr(lib, prefix + "circle_solve")
    fn.restype = c_int
    fn.argtypes = [c_int, c_uint64, vp, vp, POINTER(_abi.gb_lm_config), c_int, POINTER(_abi.gb_solve_report), vp,
                   c_int32]
    fn = getattr(lib, prefix + "vi_solve")
    fn.restype = c_int
    fn.argtypes = [c_int, c_uint64, vp, vp, c_uint64, vp, c_uint64, vp, c_uint64, vp, vp, vp, c_uint64, vp, vp, vp,
                   POINTER(_abi.gb_lm_config), c_int, POINTER(_abi.gb_solve_report), vp, c_int32]
    fn = getattr(lib, prefix + "last_error")
    fn.restype = ctypes.c_char_p
    fn.argtypes = []
    return lib


_DECLARED = set()


def device_lib():
    """libgb_bal.so with the gbg_ entry points (no CPU fallback)."""
    lib = _abi.lib()
    if "gbg" not in _DECLARED:
        _declare(lib, "gbg_")
        _DECLARED.add("gbg")
    return lib


def _check(lib, prefix, rc):
    if rc == _abi.GB_OK:
        return
    msg = getattr(lib, prefix + "last_error")().decode()
    if rc == _abi.GB_ERR_INVALID_ARGUMENT:
        raise ValueError(msg)
    raise RuntimeError(msg)


# ---------------------------------------------------------------- problems
@dataclass
class CircleProblem:
    points: np.ndarray  # (n, 2) float64
    radius: np.ndarray  # (n,)


def synthetic_circle(n: int, radius: float = 3.0, noise: float = 0.05, seed: int = 7) -> CircleProblem:
    """Points scattered around a circle (the toy's make_circle_problem shape)."""
    rng = np.random.default_rng(seed)
    th = rng.uniform(0, 2 * np.pi, n)
    r = radius + noise * rng.standard_normal(n)
    pts = np.stack([r * np.cos(th), r * np.sin(th)], axis=1) * (1 + 0.1 * rng.standard_normal((n, 1)))
    return CircleProblem(np.ascontiguousarray(pts), np.full(n, radius))


@dataclass
class ViProblem:
    poses: np.ndarray      # (K, 6) [angle-axis body->world | position]
    vbs: np.ndarray        # (K, 9) [velocity | gyro bias | accel bias]
    landmarks: np.ndarray  # (L, 3)
    st_idx: np.ndarray     # (S, 2) uint32 (pose, landmark)
    st_obs: np.ndarray     # (S, 3) (uL, vL, uR)
    cam: np.ndarray        # (5,) fx fy cx cy baseline
    imu_idx: np.ndarray    # (I, 4) uint32 (pose_i, vb_i, pose_j, vb_j)
    imu_obs: np.ndarray    # (I, 19) dp[3] dv[3] dR[9] dt pad[3]
    gravity: np.ndarray    # (3,)
    pose_fixed: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint8))

    def copy(self) -> "ViProblem":
        return ViProblem(*(np.array(getattr(self, k)) for k in
                           ("poses", "vbs", "landmarks", "st_idx", "st_obs", "cam", "imu_idx", "imu_obs", "gravity",
                            "pose_fixed")))


def rodrigues(w: np.ndarray) -> np.ndarray:
    """Rotation matrices of angle-axis vectors (gb_generic_models.hpp rotation)."""
    w = np.atleast_2d(w)
    t2 = (w * w).sum(1)
    th = np.sqrt(t2)
    small = t2 < 1e-8
    a = np.where(small, 1 - t2 * 0.5, np.cos(th))
    s = np.where(small, 1 - t2 / 6, np.sin(th) / np.where(small, 1, th))
    c = np.where(small, 0.5 - t2 / 24, (1 - np.cos(th)) / np.where(small, 1, t2))
    K = np.zeros((len(w), 3, 3))
    K[:, 0, 1], K[:, 0, 2], K[:, 1, 2] = -w[:, 2], w[:, 1], -w[:, 0]
    K[:, 1, 0], K[:, 2, 0], K[:, 2, 1] = w[:, 2], -w[:, 1], w[:, 0]
    return a[:, None, None] * np.eye(3) + s[:, None, None] * K + c[:, None, None] * np.einsum("ni,nj->nij", w, w)


def _log_so3(R: np.ndarray) -> np.ndarray:
    tr = np.clip((np.trace(R, axis1=1, axis2=2) - 1) / 2, -1, 1)
    th = np.arccos(tr)
    v = np.stack([R[:, 2, 1] - R[:, 1, 2], R[:, 0, 2] - R[:, 2, 0], R[:, 1, 0] - R[:, 0, 1]], 1)
    f = np.where(th < 1e-8, 0.5, th / (2 * np.sin(np.maximum(th, 1e-12))))
    return v * f[:, None]


def synthetic_vi(keyframes: int = 1000, landmarks: int = 20000, obs_per_kf: int = 120, dt: float = 0.1,
                 seed: int = 11) -> ViProblem:
    """EuRoC-shaped VI BA (machine hall / vicon room scale): a stereo
    camera-IMU rig flying a smooth 3-D path through a 12 x 12 x 6 m room,
    landmarks on the walls, keyframes every `dt` s with stereo observations
    (0.5 px noise) of visible landmarks, IMU preintegration edges between
    consecutive keyframes (noisy ground-truth deltas), zero biases. The
    initial estimate perturbs the ground truth; the first pose is fixed."""
    rng = np.random.default_rng(seed)
    t = np.arange(keyframes) * dt
    T = keyframes * dt
    ph = 2 * np.pi * t / T
    pos = np.stack([4 * np.sin(2 * ph), 4 * np.sin(ph), 3 + 0.8 * np.sin(3 * ph)], 1)
    vel = np.gradient(pos, dt, axis=0)
    yaw = np.arctan2(vel[:, 1], vel[:, 0])
    # body z axis = forward (camera looks along the velocity), y down
    fwd = vel / np.linalg.norm(vel, axis=1, keepdims=True)
    down = np.array([0, 0, -1.0])
    right = np.cross(down, fwd)
    right /= np.linalg.norm(right, axis=1, keepdims=True)
    dn = np.cross(fwd, right)
    Rwb = np.stack([right, dn, fwd], axis=2)  # columns: body axes in the world
    w = _log_so3(Rwb)
    del yaw
    # landmarks on the room walls
    L = landmarks
    face = rng.integers(0, 5, L)
    u, v = rng.uniform(-1, 1, L), rng.uniform(0, 1, L)
    X = np.zeros((L, 3))
    X[face == 0] = np.stack([np.full((face == 0).sum(), 6.0), 6 * u[face == 0], 6 * v[face == 0]], 1)
    X[face == 1] = np.stack([np.full((face == 1).sum(), -6.0), 6 * u[face == 1], 6 * v[face == 1]], 1)
    X[face == 2] = np.stack([6 * u[face == 2], np.full((face == 2).sum(), 6.0), 6 * v[face == 2]], 1)
    X[face == 3] = np.stack([6 * u[face == 3], np.full((face == 3).sum(), -6.0), 6 * v[face == 3]], 1)
    X[face == 4] = np.stack([6 * u[face == 4], 6 * v[face == 4] * 2 - 6, np.full((face == 4).sum(), 6.0)], 1)
    cam = np.array([458.0, 457.0, 367.0, 248.0, 0.11])
    fx, fy, cx, cy, b = cam
    st_i, st_l, st_o = [], [], []
    for k in range(keyframes):
        P = (X - pos[k]) @ Rwb[k]  # R^T (X - p)
        ok = (P[:, 2] > 0.5) & (P[:, 2] < 15)
        uL = fx * P[:, 0] / np.maximum(P[:, 2], 1e-9) + cx
        vL = fy * P[:, 1] / np.maximum(P[:, 2], 1e-9) + cy
        uR = fx * (P[:, 0] - b) / np.maximum(P[:, 2], 1e-9) + cx
        ok &= (uL > 0) & (uL < 752) & (vL > 0) & (vL < 480) & (uR > 0)
        idx = np.flatnonzero(ok)
        if len(idx) > obs_per_kf:
            idx = rng.choice(idx, obs_per_kf, replace=False)
        idx.sort()
        st_i.append(np.full(len(idx), k))
        st_l.append(idx)
        st_o.append(np.stack([uL[idx], vL[idx], uR[idx]], 1) + 0.5 * rng.standard_normal((len(idx), 3)))
    st_idx = np.stack([np.concatenate(st_i), np.concatenate(st_l)], 1).astype(np.uint32)
    st_obs = np.concatenate(st_o)
    g = np.array([0, 0, -9.81])
    I = keyframes - 1
    imu_idx = np.stack([np.arange(I), np.arange(I), np.arange(1, I + 1), np.arange(1, I + 1)], 1).astype(np.uint32)
    imu_obs = np.zeros((I, 19))
    for k in range(I):
        Ri, Rj = Rwb[k], Rwb[k + 1]
        imu_obs[k, 0:3] = Ri.T @ (pos[k + 1] - pos[k] - vel[k] * dt - 0.5 * g * dt * dt) + 0.002 * rng.standard_normal(3)
        imu_obs[k, 3:6] = Ri.T @ (vel[k + 1] - vel[k] - g * dt) + 0.005 * rng.standard_normal(3)
        dR = Ri.T @ Rj @ rodrigues(0.001 * rng.standard_normal(3))[0]
        imu_obs[k, 6:15] = dR.reshape(-1)
        imu_obs[k, 15] = dt
    poses = np.concatenate([w, pos], 1)
    vbs = np.concatenate([vel, np.zeros((keyframes, 6))], 1)
    # initial estimate
    poses0 = poses.copy()
    poses0[1:, :3] += 0.01 * rng.standard_normal((keyframes - 1, 3))
    poses0[1:, 3:] += 0.05 * rng.standard_normal((keyframes - 1, 3))
    vbs0 = vbs.copy()
    vbs0[:, :3] += 0.05 * rng.standard_normal((keyframes, 3))
    X0 = X + 0.1 * rng.standard_normal(X.shape)
    fixed = np.zeros(keyframes, np.uint8)
    fixed[0] = 1
    return ViProblem(np.ascontiguousarray(poses0), np.ascontiguousarray(vbs0), np.ascontiguousarray(X0), st_idx,
                     np.ascontiguousarray(st_obs), cam, imu_idx, imu_obs, g, fixed)


# ------------------------------------------------------------------ solves
def _prec(precision: str) -> int:
    if precision not in PREC:
        raise ValueError(f"generic path: precision pair must be fp64 or fp32, not {precision!r}")
    return PREC[precision]


def _solve(lib, prefix, call, config: LMConfig):
    c = config.to_c()
    rep = _abi.gb_solve_report()
    n = max(1, config.max_iterations)
    recs = (_abi.gb_iteration_record * n)()
    _check(lib, prefix, call(ctypes.byref(c), ctypes.byref(rep), recs, n))
    return _report(rep, recs)


def solve_circle(problem: CircleProblem, precision: str = "fp64", config: Optional[LMConfig] = None, device: int = 0,
                 lib=None, prefix: str = "gbg_", extra: int = 0) -> SolveReport:
    """Refines problem.points in place; returns the SolveReport."""
    lib = lib or device_lib()
    config = config or LMConfig()
    pts = problem.points
    assert pts.dtype == np.float64 and pts.flags.c_contiguous
    rad = np.ascontiguousarray(problem.radius, np.float64)
    fn = getattr(lib, prefix + "circle_solve")
    return _solve(lib, prefix, lambda c, r, recs, n: fn(_prec(precision), pts.shape[0], pts.ctypes.data,
                                                         rad.ctypes.data, c, device if prefix == "gbg_" else extra,
                                                         r, recs, n), config)


def solve_vi(problem: ViProblem, precision: str = "fp64", config: Optional[LMConfig] = None, device: int = 0,
             lib=None, prefix: str = "gbg_", extra: int = 0) -> SolveReport:
    """Refines problem.poses / vbs / landmarks in place; returns the SolveReport."""
    lib = lib or device_lib()
    config = config or LMConfig()
    p = problem
    for a in (p.poses, p.vbs, p.landmarks):
        assert a.dtype == np.float64 and a.flags.c_contiguous
    st_idx = np.ascontiguousarray(p.st_idx, np.uint32)
    st_obs = np.ascontiguousarray(p.st_obs, np.float64)
    imu_idx = np.ascontiguousarray(p.imu_idx, np.uint32)
    imu_obs = np.ascontiguousarray(p.imu_obs, np.float64)
    cam = np.ascontiguousarray(p.cam, np.float64)
    g = np.ascontiguousarray(p.gravity, np.float64)
    fixed = np.ascontiguousarray(p.pose_fixed, np.uint8) if len(p.pose_fixed) else None
    fn = getattr(lib, prefix + "vi_solve")
    return _solve(lib, prefix, lambda c, r, recs, n: fn(
        _prec(precision), p.poses.shape[0], p.poses.ctypes.data, None if fixed is None else fixed.ctypes.data,
        p.vbs.shape[0], p.vbs.ctypes.data, p.landmarks.shape[0], p.landmarks.ctypes.data, st_idx.shape[0],
        st_idx.ctypes.data, st_obs.ctypes.data, cam.ctypes.data, imu_idx.shape[0], imu_idx.ctypes.data,
        imu_obs.ctypes.data, g.ctypes.data, c, device if prefix == "gbg_" else extra, r, recs, n), config)
