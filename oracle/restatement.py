"""TEST INFRASTRUCTURE ONLY — numpy restatement of the reference's LM inner
loop for BAL problems (the CPU oracle).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may use
this module, and only as the checker. It restates, function by function,
/root/reference/proj/include/gopt (citations are file:line there) for the
exact graph the reference's bal::build_graph produces (one camera descriptor,
one point descriptor, one ReprojectionFactor descriptor, identity
information, Default or Huber loss):

  * sequential FP sums are reproduced with np.cumsum (left-to-right), the
    per-vertex segmented accumulations with np.add.at in incidence-item order
    (np.add.at applies repeated indices in array order), so association order
    matches the reference's single-worker loops;
  * precision pairs follow precision.hpp:72-100: FP = graph precision,
    SP = storage (bfloat16 emulated by RNE rounding of float32 bits,
    bfloat16.hpp:25-33), Arith = SP or float32 for bf16.

Pinned against the compiled reference (oracle/_ref) in
tests/test_oracle_cpu.py; parity is bit-exact for the CSR and within a few
ulps elsewhere (the LLT inverse goes through LAPACK instead of Eigen).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

# --------------------------------------------------------------- precision


def bf16_round(x: np.ndarray) -> np.ndarray:
    """bfloat16::round_from (bfloat16.hpp:25-33) -> float32 values."""
    f = np.asarray(x, np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    bias = 0x7FFF + ((u >> 16) & 1)
    r = ((u + bias) >> 16).astype(np.uint32)
    nan = np.isnan(f)
    r = np.where(nan, ((u >> 16) & 0x8000).astype(np.uint32) | 0x7FC0, r)
    return (r.astype(np.uint32) << 16).view(np.float32)


class Prec:
    """Precision pair (precision.hpp:35-100, src/experiment.cpp:153-157)."""

    def __init__(self, name: str):
        self.name = name
        self.FP = np.float64 if name == "fp64" else np.float32
        self.A = self.FP  # Arith: SP, or float for bf16
        self.bf16 = name == "fp32-bf16"

    def narrow(self, x):  # precision.hpp:86-94
        if self.bf16:
            return bf16_round(np.asarray(x, np.float32))
        return np.asarray(x, self.FP)

    @property
    def taylor(self):  # snavely.hpp:13-14
        return 1e-6 if self.FP == np.float64 else 1e-2


def seqsum(v, dtype):
    """Sequential left-to-right sum in dtype (factor_descriptor.hpp:755-759)."""
    v = np.asarray(v, dtype)
    if v.size == 0:
        return dtype(0)
    return np.cumsum(v, dtype=dtype)[-1]


# ------------------------------------------------------------ Snavely model

def rotate(w, X, P: Prec):
    """rotate_angle_axis (snavely.hpp:18-43), vectorised over rows."""
    T = P.FP
    w = np.asarray(w, T)
    X = np.asarray(X, T)
    th2 = w[:, 0] * w[:, 0] + w[:, 1] * w[:, 1] + w[:, 2] * w[:, 2]
    small = th2 < T(P.taylor)
    u = th2
    with np.errstate(all="ignore"):
        th = np.sqrt(th2)
        a = np.where(small, T(1) - u * T(0.5) + u * u * (T(1) / T(24)), np.cos(th))
        s = np.where(small, T(1) - u * (T(1) / T(6)) + u * u * (T(1) / T(120)), np.sin(th) / th)
        c = np.where(small, T(0.5) - u * (T(1) / T(24)) + u * u * (T(1) / T(720)), (T(1) - np.cos(th)) / th2)
    wx = w[:, 1] * X[:, 2] - w[:, 2] * X[:, 1]
    wy = w[:, 2] * X[:, 0] - w[:, 0] * X[:, 2]
    wz = w[:, 0] * X[:, 1] - w[:, 1] * X[:, 0]
    dot = w[:, 0] * X[:, 0] + w[:, 1] * X[:, 1] + w[:, 2] * X[:, 2]
    y0 = a * X[:, 0] + s * wx + c * dot * w[:, 0]
    y1 = a * X[:, 1] + s * wy + c * dot * w[:, 1]
    y2 = a * X[:, 2] + s * wz + c * dot * w[:, 2]
    return np.stack([y0, y1, y2], 1).astype(T)


def residual(cam, X, obs, P: Prec):
    """ReprojectionTraits::residual (adapter.hpp:58-65) -> snavely_project (snavely.hpp:48-61)."""
    T = P.FP
    p = rotate(cam[:, 0:3], X, P)
    p = p + cam[:, 3:6]
    with np.errstate(all="ignore"):
        xp = -p[:, 0] / p[:, 2]
        yp = -p[:, 1] / p[:, 2]
    n = xp * xp + yp * yp
    d = T(1) + n * (cam[:, 7] + n * cam[:, 8])
    return np.stack([cam[:, 6] * d * xp - obs[:, 0], cam[:, 6] * d * yp - obs[:, 1]], 1).astype(T)


def jacobians(cam, X, P: Prec):
    """snavely_camera_jacobian / snavely_point_jacobian via SnavelyChain
    (snavely.hpp:67-153). Returns (E,2,9), (E,2,3) at FP."""
    T = P.FP
    w = cam[:, 0:3].astype(T)
    x = X.astype(T)
    th2 = np.sum(w * w, 1)
    u = th2
    small = th2 < T(P.taylor)
    with np.errstate(all="ignore"):
        th = np.sqrt(th2)
        ca, sa = np.cos(th), np.sin(th)
        a = np.where(small, T(1) - u / T(2) + u * u / T(24), ca)
        s = np.where(small, T(1) - u / T(6) + u * u / T(120), sa / th)
        c = np.where(small, T(0.5) - u / T(24) + u * u / T(720), (T(1) - ca) / th2)
        s1 = np.where(small, -T(1) / T(3) + u / T(30), (ca - sa / th) / th2)
        c2 = np.where(small, -T(1) / T(12) + u / T(180), (sa / th - T(2) * (T(1) - ca) / th2) / th2)
    E = cam.shape[0]
    I3 = np.eye(3, dtype=T)

    def skew(v):
        z = np.zeros(E, T)
        return np.stack([np.stack([z, -v[:, 2], v[:, 1]], 1), np.stack([v[:, 2], z, -v[:, 0]], 1),
                         np.stack([-v[:, 1], v[:, 0], z], 1)], 1)

    wwT = w[:, :, None] * w[:, None, :]
    R = a[:, None, None] * I3 + s[:, None, None] * skew(w) + c[:, None, None] * wwT
    cr = np.cross(w, x)
    dt = np.sum(w * x, 1)
    Dw = (-s[:, None, None] * x[:, :, None] * w[:, None, :] + s1[:, None, None] * cr[:, :, None] * w[:, None, :]
          - s[:, None, None] * skew(x) + (c2 * dt)[:, None, None] * wwT
          + c[:, None, None] * (w[:, :, None] * x[:, None, :] + dt[:, None, None] * I3))
    P3 = np.einsum("eij,ej->ei", R, x) + cam[:, 3:6]
    with np.errstate(all="ignore"):
        iz = T(1) / P3[:, 2]
    p = np.stack([-P3[:, 0] * iz, -P3[:, 1] * iz], 1)
    n = np.sum(p * p, 1)
    f, k1, k2 = cam[:, 6], cam[:, 7], cam[:, 8]
    dist = T(1) + n * (k1 + n * k2)
    z = np.zeros(E, T)
    dpdP = np.stack([np.stack([-iz, z, P3[:, 0] * iz * iz], 1), np.stack([z, -iz, P3[:, 1] * iz * iz], 1)], 1)
    dudp = f[:, None, None] * (dist[:, None, None] * np.eye(2, dtype=T)
                               + (T(2) * (k1 + T(2) * k2 * n))[:, None, None] * p[:, :, None] * p[:, None, :])
    U = np.einsum("eij,ejk->eik", dudp, dpdP)
    Jc = np.zeros((E, 2, 9), T)
    Jc[:, :, 0:3] = np.einsum("eij,ejk->eik", U, Dw)
    Jc[:, :, 3:6] = U
    Jc[:, :, 6] = dist[:, None] * p
    Jc[:, :, 7] = (f * n)[:, None] * p
    Jc[:, :, 8] = (f * n * n)[:, None] * p
    Jp = np.einsum("eij,ejk->eik", U, R)
    return Jc.astype(T), Jp.astype(T)


def loss(kind, delta, s, T):
    """loss_value / loss_weight (loss.hpp:25-40)."""
    if kind == "default":
        return s.astype(T), np.ones_like(s, dtype=T)
    d2 = T(delta) * T(delta)
    with np.errstate(all="ignore"):
        val = np.where(s <= d2, s, T(2) * T(delta) * np.sqrt(s) - d2).astype(T)
        w = np.where(s <= d2, T(1), T(delta) / np.sqrt(s)).astype(T)
    return val, w


# ------------------------------------------------------------------- graph

@dataclass
class Graph:
    """bal::build_graph (adapter.hpp:106-143) + Graph::activate (graph.hpp:59-83)."""
    P: Prec
    cams: np.ndarray
    pts: np.ndarray
    cam_idx: np.ndarray
    pt_idx: np.ndarray
    obs: np.ndarray
    cam_fixed: np.ndarray
    pt_fixed: np.ndarray
    levels: np.ndarray
    loss_kind: str = "default"
    delta: float = 1.0
    dynamic: bool = False
    # activation products
    active: np.ndarray = field(default=None)
    cam_col: np.ndarray = field(default=None)
    pt_col: np.ndarray = field(default=None)
    N: int = 0
    inc: list = field(default=None)


def build_graph(problem, precision="fp64", diff_mode="analytic", huber_delta=None, cam_fixed=None,
                pt_fixed=None, levels=None) -> Graph:
    P = Prec(precision)
    T = P.FP
    nc, np_ = problem.cameras.shape[0], problem.points.shape[0]
    ne = problem.camera_index.shape[0]
    return Graph(P, problem.cameras.astype(T).copy(), problem.points.astype(T).copy(),
                 problem.camera_index.astype(np.int64), problem.point_index.astype(np.int64),
                 problem.observations.astype(T), np.zeros(nc, bool) if cam_fixed is None else np.asarray(cam_fixed, bool),
                 np.zeros(np_, bool) if pt_fixed is None else np.asarray(pt_fixed, bool),
                 np.zeros(ne, np.int64) if levels is None else np.asarray(levels, np.int64),
                 "huber" if huber_delta is not None else "default", 1.0 if huber_delta is None else huber_delta,
                 diff_mode == "dynamic")


def incidence(nvert, vert_of_a, fixed):
    """FactorDescriptor::build_incidence (factor_descriptor.hpp:710-753)."""
    free_a = ~fixed[vert_of_a]
    counts = np.bincount(vert_of_a[free_a], minlength=nvert)
    vos = np.nonzero(counts)[0].astype(np.uint64)
    offsets = np.concatenate([[0], np.cumsum(counts[vos.astype(np.int64)])]).astype(np.uint64)
    a_idx = np.nonzero(free_a)[0]
    order = np.argsort(vert_of_a[a_idx], kind="stable")
    items = a_idx[order].astype(np.uint32)
    return vos, offsets, items


def activate(g: Graph, level: int):
    g.active = np.nonzero(g.levels <= level)[0]  # factor_descriptor.hpp:255-257
    nc, np_ = g.cams.shape[0], g.pts.shape[0]
    g.cam_col = np.full(nc, -1, np.int64)  # vertex_descriptor.hpp:115-126, cameras first
    fc = np.nonzero(~g.cam_fixed)[0]
    g.cam_col[fc] = 9 * np.arange(fc.size)
    g.pt_col = np.full(np_, -1, np.int64)
    fp = np.nonzero(~g.pt_fixed)[0]
    g.pt_col[fp] = 9 * fc.size + 3 * np.arange(fp.size)
    g.N = 9 * fc.size + 3 * fp.size
    ca = g.cam_idx[g.active]
    pa = g.pt_idx[g.active]
    g.inc = [incidence(nc, ca, g.cam_fixed), incidence(np_, pa, g.pt_fixed)]


def eval_chi_terms(g: Graph, raw=False):
    """evaluate_chi2 / raw_residual_sqnorm terms (factor_descriptor.hpp:294-320)."""
    T = g.P.FP
    a = g.active
    r = residual(g.cams[g.cam_idx[a]], g.pts[g.pt_idx[a]], g.obs[a], g.P)
    s = (r[:, 0] * r[:, 0] + r[:, 1] * r[:, 1]).astype(T)
    if raw:
        return s
    return loss(g.loss_kind, g.delta, s, T)[0]


class LinearSystem:
    """LinearSystem<FP,SP> (linear_system.hpp:34-235) for a BAL graph."""

    def __init__(self, g: Graph, clamp_min=1e-6, clamp_max=1e32, damping="after_scaling"):
        self.g = g
        self.cmin, self.cmax = clamp_min, clamp_max
        self.before = damping == "before_scaling"
        self.fallbacks = 0

    # factor_descriptor.hpp:662-684: per-factor blocks at FP, stored at SP
    def _blocks(self):
        g, P = self.g, self.g.P
        a = g.active
        Jc, Jp = jacobians(g.cams[g.cam_idx[a]], g.pts[g.pt_idx[a]], P)
        if not g.dynamic:
            Jc, Jp = P.narrow(Jc).astype(P.FP), P.narrow(Jp).astype(P.FP)
        return Jc, Jp

    def linearize(self):
        """linear_system.hpp:67-82 with factor_descriptor.hpp:272-292, 322-370."""
        g, P = self.g, self.g.P
        T = P.FP
        a = g.active
        r = residual(g.cams[g.cam_idx[a]], g.pts[g.pt_idx[a]], g.obs[a], P)
        s = (r[:, 0] * r[:, 0] + r[:, 1] * r[:, 1]).astype(T)
        terms, w = loss(g.loss_kind, g.delta, s, T)
        chi = seqsum(terms, T)
        self.w = w
        self.wr = (w[:, None] * r).astype(T)
        self.Jc, self.Jp = self._blocks()
        N = g.N
        self.b = np.zeros(N, T)
        self.diag = np.zeros(N, T)
        for which, (vos, off, items) in enumerate(g.inc):
            J = self.Jc if which == 0 else self.Jp
            dim = 9 if which == 0 else 3
            it = items.astype(np.int64)
            vert = (g.cam_idx if which == 0 else g.pt_idx)[g.active[it]]
            col = (g.cam_col if which == 0 else g.pt_col)[vert]
            Jb = J[it]
            bb = (Jb[:, 0, :] * self.wr[it, 0:1] + Jb[:, 1, :] * self.wr[it, 1:2]).astype(T)
            dd = (self.w[it, None] * (Jb[:, 0, :] * Jb[:, 0, :] + Jb[:, 1, :] * Jb[:, 1, :])).astype(T)
            cols = (col[:, None] + np.arange(dim)[None, :]).reshape(-1)
            np.add.at(self.b, cols, bb.reshape(-1))
            np.add.at(self.diag, cols, dd.reshape(-1))
        self.clamped = np.clip(self.diag, T(self.cmin), T(self.cmax)).astype(T)
        self.D = (T(1) / np.sqrt(self.clamped)).astype(T)
        self.finite = bool(np.isfinite(chi) and np.all(np.isfinite(self.b)) and np.all(np.isfinite(self.diag)))
        return chi

    def initialize_damping(self, tau):
        """linear_system.hpp:94-99."""
        T = self.g.P.FP
        if self.g.N == 0:
            return T(tau)
        return T(tau) * np.max(self.D * self.D * self.clamped)

    def hvp(self, v, lam):
        """linear_system.hpp:104-115, hvp_forward :372-407, hvp_scatter :409-433."""
        g, P = self.g, self.g.P
        A = P.A
        T = P.FP
        damp = (A(T(lam) * self.D * self.D) if self.before else A(T(lam)) * np.ones(g.N, A)).astype(A)
        out = (damp * v.astype(A)).astype(A)
        if self.g.dynamic:
            Jc, Jp = self._blocks()
        else:
            Jc, Jp = self.Jc, self.Jp
        Jc, Jp = Jc.astype(A), Jp.astype(A)
        a = g.active
        Da = self.D.astype(A)
        u = np.zeros((a.size, 2), A)
        for which in (0, 1):
            vert = (g.cam_idx if which == 0 else g.pt_idx)[a]
            col = (g.cam_col if which == 0 else g.pt_col)[vert]
            dim = 9 if which == 0 else 3
            ok = col >= 0
            cols = np.where(ok[:, None], col[:, None] + np.arange(dim)[None, :], 0)
            vt = np.where(ok[:, None], Da[cols] * v.astype(A)[cols], A(0)).astype(A)
            J = Jc if which == 0 else Jp
            acc = np.zeros((a.size, 2), A)
            for c in range(dim):  # sequential over columns, as in the reference
                acc = (acc + J[:, :, c] * vt[:, c:c + 1]).astype(A)
            u = (u + acc).astype(A)
        q = (self.w.astype(A)[:, None] * u).astype(A)
        for which, (vos, off, items) in enumerate(g.inc):
            it = items.astype(np.int64)
            vert = (g.cam_idx if which == 0 else g.pt_idx)[a[it]]
            col = (g.cam_col if which == 0 else g.pt_col)[vert]
            dim = 9 if which == 0 else 3
            J = (Jc if which == 0 else Jp)[it]
            acc = (J[:, 0, :] * q[it, 0:1] + J[:, 1, :] * q[it, 1:2]).astype(A)
            cols = (col[:, None] + np.arange(dim)[None, :])
            np.add.at(out, cols.reshape(-1), (Da[cols] * acc).astype(A).reshape(-1))
        return out

    def build_preconditioner(self, lam):
        """linear_system.hpp:120-160 with accumulate_precond_blocks factor_descriptor.hpp:435-482."""
        g = self.g
        T = g.P.FP
        a = g.active
        blocks = []
        self.fallbacks = 0
        for which, (vos, off, items) in enumerate(g.inc):
            dim = 9 if which == 0 else 3
            nfree = int(np.sum(~(g.cam_fixed if which == 0 else g.pt_fixed)))
            B = np.zeros((nfree, dim, dim), T)
            it = items.astype(np.int64)
            vert = (g.cam_idx if which == 0 else g.pt_idx)[a[it]]
            colv = (g.cam_col if which == 0 else g.pt_col)[vert]
            base = 0 if which == 0 else 9 * int(np.sum(~g.cam_fixed))
            bi = (colv - base) // dim
            J = (self.Jc if which == 0 else self.Jp)[it] if not g.dynamic else self._blocks()[which][it]
            cols = colv[:, None] + np.arange(dim)[None, :]
            Js = (J * self.D[cols][:, None, :]).astype(T)
            contrib = (self.w[it, None, None] * np.einsum("eri,erj->eij", Js, Js)).astype(T)
            np.add.at(B, bi, contrib)
            cols_all = base + dim * np.arange(nfree)[:, None] + np.arange(dim)[None, :]
            damp = T(lam) * self.D[cols_all] * self.D[cols_all] if self.before else np.full((nfree, dim), T(lam))
            B[:, np.arange(dim), np.arange(dim)] += damp
            inv = np.zeros_like(B)
            for k in range(nfree):
                try:
                    L = np.linalg.cholesky(B[k].astype(np.float64))
                    Li = np.linalg.inv(L)
                    m = (Li.T @ Li).astype(T)
                    if np.all(np.isfinite(m)):
                        inv[k] = m
                        continue
                except np.linalg.LinAlgError:
                    pass
                self.fallbacks += 1
                d = np.clip(np.diag(B[k]), T(self.cmin), T(self.cmax))
                inv[k] = np.diag(T(1) / d)
            blocks.append(inv)
        self.blocks = blocks
        return np.concatenate([blocks[0].reshape(-1), blocks[1].reshape(-1)])

    def apply_preconditioner(self, r):
        """linear_system.hpp:164-180."""
        P = self.g.P
        T = P.FP
        nfc = self.blocks[0].shape[0]
        z = np.empty(self.g.N, T)
        rc = r[: 9 * nfc].astype(T).reshape(nfc, 9)
        z[: 9 * nfc] = np.einsum("kij,kj->ki", self.blocks[0], rc).reshape(-1)
        rp = r[9 * nfc:].astype(T).reshape(-1, 3)
        z[9 * nfc:] = np.einsum("kij,kj->ki", self.blocks[1], rp).reshape(-1)
        return P.narrow(z)

    def solve_step(self, lam, pcg):
        """linear_system.hpp:185-207."""
        T = self.g.P.FP
        self.build_preconditioner(lam)
        rhs = (-self.D * self.b).astype(T)
        x, stats = pcg_solve(lambda v: self.hvp(v, lam), self.apply_preconditioner, rhs, pcg, self.g.P)
        damp = T(lam) * self.D * self.D if self.before else T(lam)
        pred = seqsum(x * (damp * x + rhs), T)
        dx = (self.D * x).astype(T)
        return dx, stats, pred, bool(np.all(np.isfinite(dx)))


def pcg_solve(A, M, rhs, cfg, P: Prec):
    """pcg_solve (pcg.hpp:34-105)."""
    T = P.FP
    n = rhs.size
    stats = dict(iterations=0, final_relative_residual=0.0, converged=False)
    nrm = np.sqrt(seqsum(rhs * rhs, T))
    if not nrm > 0:
        stats["converged"] = bool(np.isfinite(nrm))
        return np.zeros(n, T), stats
    scale = T(1) / nrm if cfg["normalize_rhs"] else T(1)
    dot = lambda a, b: seqsum(a.astype(T) * b.astype(T), T)  # noqa: E731
    x = P.narrow(np.zeros(n, T))
    r = P.narrow(rhs * scale)
    z = M(r)
    p = z.copy()
    ref = T(1) if cfg["normalize_rhs"] else nrm
    rho = dot(r, z)
    res = np.sqrt(dot(r, r))
    stats["final_relative_residual"] = float(res / ref)
    while stats["iterations"] < cfg["max_iterations"]:
        ap = P.narrow(A(p))
        pap = dot(p, ap)
        if not (pap > 0) or not np.isfinite(pap):
            stats["converged"] = False
            break
        alpha = rho / pap
        x = P.narrow(x.astype(T) + alpha * p.astype(T))
        r = P.narrow(r.astype(T) - alpha * ap.astype(T))
        stats["iterations"] += 1
        res = np.sqrt(dot(r, r))
        stats["final_relative_residual"] = float(res / ref)
        if not math.isfinite(stats["final_relative_residual"]):
            stats["converged"] = False
            break
        if res <= T(cfg["tolerance"]) * ref:
            stats["converged"] = True
            break
        z = M(r)
        rho_next = dot(r, z)
        beta = rho_next / rho
        rho = rho_next
        p = P.narrow(z.astype(T) + beta * p.astype(T))
    unscale = nrm if cfg["normalize_rhs"] else T(1)
    return (x.astype(T) * unscale).astype(T), stats


TERMS = ["max_iterations", "tolerance_reached", "gradient_small", "damping_overflow", "non_finite_linearization",
         "no_free_parameters"]


def levenberg_marquardt(g: Graph, cfg: dict):
    """levenberg_marquardt (levenberg_marquardt.hpp:115-224); update_damping :88-98.
    cfg keys mirror LMConfig (max_iterations, tolerance, level, tau, pcg{...},
    use_rejection_guard, refresh_on_reject, lambda_max, gradient_tolerance,
    clamp_min, clamp_max, damping). Refines g.cams / g.pts in place."""
    T = g.P.FP
    activate(g, cfg.get("level", 0))
    ls = LinearSystem(g, cfg.get("clamp_min", 1e-6), cfg.get("clamp_max", 1e32), cfg.get("damping", "after_scaling"))
    chi2 = ls.linearize()
    if not np.isfinite(chi2):
        raise RuntimeError("levenberg_marquardt: non-finite chi^2 at the initial parameters")
    rep = dict(initial_chi2=float(chi2), final_chi2=float(chi2), accepted_steps=0, termination="max_iterations",
               iterations=[])
    if g.N == 0:
        rep["termination"] = "no_free_parameters"
        return rep
    lam = ls.initialize_damping(cfg.get("tau", 1e-4))
    nu = T(2)
    pcg = cfg["pcg"]
    for it in range(1, cfg["max_iterations"] + 1):
        rec = dict(iteration=it, chi2_before=float(chi2), lambda_=float(lam), accepted=False, pcg_iterations=0,
                   low_quality_step=False)
        if not ls.finite:
            rec["chi2_after"] = rec["chi2_before"]
            rep["iterations"].append(rec)
            rep["termination"] = "non_finite_linearization"
            break
        if np.max(np.abs(ls.b)) < T(cfg.get("gradient_tolerance", 1e-12)):
            rec["chi2_after"] = rec["chi2_before"]
            rep["iterations"].append(rec)
            rep["termination"] = "gradient_small"
            break
        dx, stats, pred, finite = ls.solve_step(lam, pcg)
        rec["pcg_iterations"] = stats["iterations"]
        rec["pcg_converged"] = stats["converged"]
        rec["pcg_relative_residual"] = stats["final_relative_residual"]
        rec["precond_fallback_blocks"] = ls.fallbacks
        if cfg.get("use_rejection_guard", True) and not stats["converged"] and \
                stats["final_relative_residual"] > pcg["rejection_ratio"] * pcg["tolerance"]:
            rec["low_quality_step"] = True
            lam = T(lam * nu)
        snap = (g.cams.copy(), g.pts.copy())
        chi_new = T(np.nan)
        if finite:
            fc = g.cam_col >= 0
            g.cams[fc] = (g.cams[fc] + dx[g.cam_col[fc][:, None] + np.arange(9)]).astype(T)
            fp = g.pt_col >= 0
            g.pts[fp] = (g.pts[fp] + dx[g.pt_col[fp][:, None] + np.arange(3)]).astype(T)
            chi_new = seqsum(eval_chi_terms(g), T)
        rec["chi2_after"] = float(chi_new)
        accepted = bool(np.isfinite(chi_new) and chi_new < chi2)
        rec["accepted"] = accepted
        rel = T(0)
        if accepted:
            rep["accepted_steps"] += 1
            gain = (chi2 - chi_new) / pred if pred > 0 else T(np.inf)
            gg = T(2) * gain - T(1)
            lam = T(lam * max(T(1) / T(3), T(1) - gg * gg * gg))
            nu = T(2)
            rel = (chi2 - chi_new) / chi2
            chi2 = ls.linearize()
            rep["final_chi2"] = float(chi2)
        else:
            if finite:
                g.cams, g.pts = snap
            lam = T(lam * nu)
            nu = T(nu * 2)
            if cfg.get("refresh_on_reject", False):
                ls.linearize()
        rep["iterations"].append(rec)
        if accepted and float(rel) < cfg.get("tolerance", 1e-6):
            rep["termination"] = "tolerance_reached"
            break
        if float(lam) > cfg.get("lambda_max", 1e32):
            rep["termination"] = "damping_overflow"
            break
    return rep


def lm_config(max_iterations=50, pcg_iterations=10, **kw):
    """BAL parity config (tests/acceptance.cpp:69-80) as a restatement dict."""
    cfg = dict(max_iterations=max_iterations, tolerance=1e-6, level=0, tau=1e-4,
               pcg=dict(max_iterations=pcg_iterations, tolerance=1e-6, rejection_ratio=10.0, normalize_rhs=True))
    cfg.update(kw)
    return cfg


def update_damping(lam, nu, accepted, gain):
    """Nielsen schedule (levenberg_marquardt.hpp:88-98)."""
    if accepted:
        g = 2.0 * gain - 1.0
        return lam * max(1.0 / 3.0, 1.0 - g * g * g), 2.0
    return lam * nu, nu * 2.0


def project(camera, point, precision="fp64"):
    """snavely_project for one camera/point (snavely.hpp:48-61)."""
    P = Prec(precision)
    c = np.asarray(camera, P.FP)[None, :]
    x = np.asarray(point, P.FP)[None, :]
    return residual(c, x, np.zeros((1, 2), P.FP), P)[0]


# ------------------------------------------------------------ Schur mode
# Not in the reference (SPEC.md:164, 366 non-goal; PAPER.md:561 future work):
# this is the CPU statement of the device Schur-complement solver mode
# (SURVEY.md §8 f-1), checked against a dense oracle in the tests. On the
# scaled, damped system A = D H D + Lambda (linear_system.hpp:104-115) with
# camera (c) / point (p) blocks:
#   S = A_cc - A_cp A_pp^-1 A_pc,  r_c = rhs_c - A_cp A_pp^-1 rhs_p
#   S x_c = r_c by pcg_solve with block-Jacobi on S's camera blocks,
#   x_p = A_pp^-1 (rhs_p - A_pc x_c); pred and dx as in solve_step.
class SchurSystem:
    def __init__(self, ls: LinearSystem):
        self.ls = ls
        g = ls.g
        a = g.active
        self.cam = g.cam_idx[a]
        self.pt = g.pt_idx[a]
        nfc = int(np.sum(~g.cam_fixed))
        self.nfc = nfc
        self.ccol = g.cam_col[self.cam]
        self.pcol = g.pt_col[self.pt]

    def _parts(self, lam):
        ls, g = self.ls, self.ls.g
        T = g.P.FP
        D = ls.D
        Jc, Jp = ls.Jc.astype(T), ls.Jp.astype(T)
        ok_c = self.ccol >= 0
        ok_p = self.pcol >= 0
        cc = np.where(ok_c[:, None], self.ccol[:, None] + np.arange(9), 0)
        pc = np.where(ok_p[:, None], self.pcol[:, None] + np.arange(3), 0)
        Jtc = np.where(ok_c[:, None, None], Jc * D[cc][:, None, :], 0)
        Jtp = np.where(ok_p[:, None, None], Jp * D[pc][:, None, :], 0)
        w = ls.w.astype(T)
        lamv = (T(lam) * D * D) if ls.before else np.full(g.N, T(lam))
        N = g.N
        npf = (N - 9 * self.nfc) // 3
        App = np.zeros((npf, 3, 3), T)
        pidx = np.where(ok_p, (self.pcol - 9 * self.nfc) // 3, 0)
        np.add.at(App, pidx[ok_p], (w[:, None, None] * np.einsum("eri,erj->eij", Jtp, Jtp))[ok_p])
        App[:, np.arange(3), np.arange(3)] += lamv[9 * self.nfc:].reshape(npf, 3)
        Ainv = np.linalg.inv(App.astype(np.float64)).astype(T)
        return Jtc, Jtp, w, lamv, pidx, ok_c, ok_p, Ainv, cc, pc

    def operator(self, lam):
        Jtc, Jtp, w, lamv, pidx, ok_c, ok_p, Ainv, cc, pc = self._parts(lam)
        nfc, T = self.nfc, self.ls.g.P.FP

        def S(v):  # camera-sized
            vv = np.zeros(self.ls.g.N, T)
            vv[: 9 * nfc] = v
            u = np.einsum("erc,ec->er", Jtc, vv[cc] * ok_c[:, None])
            q = w[:, None] * u
            y = np.zeros((Ainv.shape[0], 3), T)
            np.add.at(y, pidx[ok_p], np.einsum("erc,er->ec", Jtp, q)[ok_p])
            z = np.einsum("pij,pj->pi", Ainv, y)
            u2 = np.einsum("erc,ec->er", Jtp, z[pidx] * ok_p[:, None])
            g = np.einsum("erc,er->ec", Jtc, w[:, None] * (u - u2))
            out = lamv[: 9 * nfc] * v
            np.add.at(out, cc[ok_c].ravel(), g[ok_c].ravel())
            return out

        return S

    def solve_step(self, lam, pcg):
        ls, g = self.ls, self.ls.g
        T = g.P.FP
        Jtc, Jtp, w, lamv, pidx, ok_c, ok_p, Ainv, cc, pc = self._parts(lam)
        nfc = self.nfc
        rhs = (-ls.D * ls.b).astype(T)
        rc, rp = rhs[: 9 * nfc], rhs[9 * nfc:].reshape(-1, 3)
        zp = np.einsum("pij,pj->pi", Ainv, rp)
        u2 = np.einsum("erc,ec->er", Jtp, zp[pidx] * ok_p[:, None])
        gc = np.einsum("erc,er->ec", Jtc, w[:, None] * u2)
        r = rc.copy()
        np.add.at(r, cc[ok_c].ravel(), -gc[ok_c].ravel())
        # block-Jacobi of S: A_cc(c) - sum_e B_e A_pp^-1 B_e^T, B_e = w Jtc^T Jtp
        Scc = np.zeros((nfc, 9, 9), T)
        cidx = np.where(ok_c, self.ccol // 9, 0)
        np.add.at(Scc, cidx[ok_c], (w[:, None, None] * np.einsum("eri,erj->eij", Jtc, Jtc))[ok_c])
        B = w[:, None, None] * np.einsum("eri,erj->eij", Jtc, Jtp)
        corr = np.einsum("eij,ejk,elk->eil", B, Ainv[pidx], B)
        sel = ok_c & ok_p
        np.add.at(Scc, cidx[sel], -corr[sel])
        Scc[:, np.arange(9), np.arange(9)] += lamv[: 9 * nfc].reshape(nfc, 9)
        Minv = np.linalg.inv(Scc.astype(np.float64)).astype(T)

        def M(v):
            return g.P.narrow(np.einsum("kij,kj->ki", Minv, v.astype(T).reshape(nfc, 9)).reshape(-1))

        xc, stats = pcg_solve(self.operator(lam), M, r, pcg, g.P)
        xx = np.zeros(g.N, T)
        xx[: 9 * nfc] = xc
        u = np.einsum("erc,ec->er", Jtc, xx[cc] * ok_c[:, None])
        y = np.zeros_like(rp)
        np.add.at(y, pidx[ok_p], np.einsum("erc,er->ec", Jtp, w[:, None] * u)[ok_p])
        xp = np.einsum("pij,pj->pi", Ainv, rp - y)
        x = np.concatenate([xc, xp.reshape(-1)]).astype(T)
        damp = T(lam) * ls.D * ls.D if ls.before else T(lam)
        pred = seqsum(x * (damp * x + rhs), T)
        dx = (ls.D * x).astype(T)
        return dx, stats, pred, bool(np.all(np.isfinite(dx)))

    def dense(self, lam):
        """Dense A, S, r_c and the exact Schur solution (the dense oracle)."""
        ls, g = self.ls, self.ls.g
        N, nfc = g.N, self.nfc
        A = np.zeros((N, N))
        I = np.eye(N)
        for k in range(N):
            A[:, k] = ls.hvp(I[k].astype(g.P.FP), lam)
        rhs = -ls.D * ls.b
        c = slice(0, 9 * nfc)
        p = slice(9 * nfc, N)
        Spp = np.linalg.inv(A[p, p])
        S = A[c, c] - A[c, p] @ Spp @ A[p, c]
        r = rhs[c] - A[c, p] @ Spp @ rhs[p]
        xc = np.linalg.solve(S, r)
        xp = Spp @ (rhs[p] - A[p, c] @ xc)
        return A, S, r, np.concatenate([xc, xp]), rhs
