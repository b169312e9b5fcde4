"""Host-side mirror of the reference's BAL API over the C ABI.

Same names, argument meaning and error behaviour as the reference C++ API so
that parity tests read like the reference's own tests:

  reference (C++, /root/reference/proj)                 here
  ----------------------------------------------------  -------------------------------
  bal::BALProblem           bal/problem.hpp:25-40       BALProblem
  bal::parse_bal_text / serialize_bal_text              parse_bal_text / serialize_bal_text
  bal::build_graph<FP,SP>   bal/adapter.hpp:106-143     build_graph(problem, precision, mode)
  BalGraph::mse             bal/adapter.hpp:95-99       BalGraph.mse()
  Graph::total_error        graph.hpp:99-104            BalGraph.total_error(level)
  VertexDescriptor::set_fixed vertex_descriptor.hpp:80  BalGraph.set_fixed(...)
  FactorDescriptor::set_level factor_descriptor.hpp:222 BalGraph.set_levels(...)
  LMConfig / PCGConfig      levenberg_marquardt.hpp:15  LMConfig / PCGConfig
  levenberg_marquardt       levenberg_marquardt.hpp:115 levenberg_marquardt(graph, config)
  SolveReport / IterationRecord :49-83                  SolveReport / IterationRecord
  LinearSystem accessors    linear_system.hpp:44-216    BalGraph.ls_* (parity surface)

Errors raise the Python counterpart of the reference exception
(ValueError <- std::invalid_argument, IndexError <- std::out_of_range,
LogicError <- std::logic_error, RuntimeError <- std::runtime_error).
The device path never falls back to the CPU.
"""
from __future__ import annotations

import ctypes
import dataclasses
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _abi

PRECISIONS = {"fp64": _abi.GB_FP64, "fp32": _abi.GB_FP32, "fp32-bf16": _abi.GB_FP32_BF16}
MODES = {"analytic": _abi.GB_ANALYTIC, "auto": _abi.GB_AUTO, "dynamic": _abi.GB_DYNAMIC}


class LogicError(RuntimeError):
    """std::logic_error counterpart."""


class DeviceError(RuntimeError):
    """CUDA failure or no device (no reference counterpart)."""


def dtypes(precision: str):
    """(FP, SP, Arith) numpy dtypes of a precision pair (precision.hpp:72-81)."""
    if precision == "fp64":
        return np.float64, np.float64, np.float64
    if precision == "fp32":
        return np.float32, np.float32, np.float32
    if precision == "fp32-bf16":
        return np.float32, np.uint16, np.float32
    raise ValueError(f"invalid precision pair: {precision}")


def bf16_bits(x) -> np.ndarray:
    """float -> bfloat16 storage bits, RNE with the quiet-NaN encoding of
    bfloat16::round_from (bfloat16.hpp:25-33)."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)
    nan = np.isnan(np.asarray(x, dtype=np.float32))
    r[nan] = (((u[nan] >> 16) & 0x8000) | 0x7FC0).astype(np.uint16)
    return r


def _to_storage(v, sp):
    """Values in the storage type SP (bf16 storage = uint16 bits)."""
    if sp is np.uint16 and np.asarray(v).dtype != np.uint16:
        return bf16_bits(v)
    return np.ascontiguousarray(v, dtype=sp)


# --------------------------------------------------------------------- configs
@dataclass
class PCGConfig:
    """pcg.hpp:12-17."""
    max_iterations: int = 50
    tolerance: float = 1e-6
    rejection_ratio: float = 10.0
    normalize_rhs: bool = True

    def to_c(self) -> _abi.gb_pcg_config:
        return _abi.gb_pcg_config(self.max_iterations, self.tolerance, self.rejection_ratio, int(self.normalize_rhs))


@dataclass
class LMConfig:
    """levenberg_marquardt.hpp:15-26 (+ LinearSystemOptions, linear_system.hpp:15-19)."""
    max_iterations: int = 10
    tolerance: float = 1e-6
    level: int = 0
    tau: float = 1e-4
    pcg: PCGConfig = field(default_factory=PCGConfig)
    clamp_min: float = 1e-6
    clamp_max: float = 1e32
    damping: str = "after_scaling"
    use_rejection_guard: bool = True
    refresh_on_reject: bool = False
    lambda_max: float = 1e32
    gradient_tolerance: float = 1e-12

    def to_c(self) -> _abi.gb_lm_config:
        c = _abi.gb_lm_config()
        c.max_iterations = self.max_iterations
        c.tolerance = self.tolerance
        c.level = self.level
        c.tau = self.tau
        c.pcg = self.pcg.to_c()
        c.clamp_min = self.clamp_min
        c.clamp_max = self.clamp_max
        c.damping = _abi.GB_DAMPING_BEFORE_SCALING if self.damping == "before_scaling" else _abi.GB_DAMPING_AFTER_SCALING
        c.use_rejection_guard = int(self.use_rejection_guard)
        c.refresh_on_reject = int(self.refresh_on_reject)
        c.lambda_max = self.lambda_max
        c.gradient_tolerance = self.gradient_tolerance
        return c


@dataclass
class IterationRecord:
    iteration: int
    chi2_before: float
    chi2_after: float
    lambda_: float
    pcg_iterations: int
    pcg_converged: bool
    pcg_relative_residual: float
    low_quality_step: bool
    precond_fallback_blocks: int
    accepted: bool
    wall_seconds: float


@dataclass
class SolveReport:
    iterations: List[IterationRecord]
    initial_chi2: float
    final_chi2: float
    accepted_steps: int
    termination: str
    total_seconds: float
    free_dims: int
    residual_dims: int
    active_factors: int
    memory: dict
    setup_seconds: float = 0.0
    h2d_bytes: float = 0.0
    d2h_bytes: float = 0.0

    def to_dict(self) -> dict:
        d = dataclasses.asdict(self)
        for it in d["iterations"]:
            it["lambda"] = it.pop("lambda_")
        return d

    def to_c(self):
        """(gb_solve_report, gb_iteration_record[n]) of this report."""
        r = _abi.gb_solve_report()
        r.initial_chi2, r.final_chi2 = self.initial_chi2, self.final_chi2
        r.accepted_steps = self.accepted_steps
        r.termination = _abi.TERMINATION_NAMES.index(self.termination)
        r.total_seconds = self.total_seconds
        r.free_dims, r.residual_dims, r.active_factors = self.free_dims, self.residual_dims, self.active_factors
        for k in ("jacobian_bytes", "preconditioner_bytes", "workspace_bytes", "graph_bytes"):
            setattr(r.memory, k, int(self.memory[k]))
        n = len(self.iterations)
        r.iterations_run = n
        recs = (_abi.gb_iteration_record * max(1, n))()
        for c, it in zip(recs, self.iterations):
            c.iteration, c.chi2_before, c.chi2_after, c.lambda_ = it.iteration, it.chi2_before, it.chi2_after, it.lambda_
            c.pcg_iterations, c.pcg_converged = it.pcg_iterations, int(it.pcg_converged)
            c.pcg_relative_residual, c.low_quality_step = it.pcg_relative_residual, int(it.low_quality_step)
            c.precond_fallback_blocks, c.accepted, c.wall_seconds = (it.precond_fallback_blocks, int(it.accepted),
                                                                     it.wall_seconds)
        return r, recs

    def _wire(self, name: str) -> str:
        r, recs = self.to_c()
        fn = getattr(_abi.lib(), "gb_report_" + name)
        need = ctypes.c_uint64()
        Backend(_abi.lib(), "gb_").check(fn(ctypes.byref(r), recs, len(self.iterations), None, 0, ctypes.byref(need)))
        buf = ctypes.create_string_buffer(need.value)
        Backend(_abi.lib(), "gb_").check(fn(ctypes.byref(r), recs, len(self.iterations), buf, need.value, None))
        return buf.value.decode()

    def to_json(self) -> str:
        """gopt::to_json(report).dump() (report.hpp:32-47), byte for byte."""
        return self._wire("json")

    def to_csv(self) -> str:
        """gopt::to_csv(report) (report.hpp:51-71), byte for byte."""
        return self._wire("csv")


# ---------------------------------------------------------------- BAL problem
@dataclass
class BALProblem:
    """bal/problem.hpp:25-40 (binary64 values)."""
    cameras: np.ndarray  # (nc, 9) float64
    points: np.ndarray  # (np, 3) float64
    camera_index: np.ndarray  # (ne,) uint32
    point_index: np.ndarray  # (ne,) uint32
    observations: np.ndarray  # (ne, 2) float64

    @property
    def num_cameras(self) -> int:
        return int(self.cameras.shape[0])

    @property
    def num_points(self) -> int:
        return int(self.points.shape[0])

    @property
    def num_observations(self) -> int:
        return int(self.camera_index.shape[0])

    def copy(self) -> "BALProblem":
        return BALProblem(self.cameras.copy(), self.points.copy(), self.camera_index.copy(), self.point_index.copy(),
                          self.observations.copy())


def synthetic_bal(num_cameras: int, num_points: int, num_observations: int, seed: int = 42,
                  camera_stride: int = 0, zipf: float = 0.0) -> BALProblem:
    """Deterministic BAL-shaped problem (gb_synthetic_bal)."""
    nc, np_, ne = int(num_cameras), int(num_points), int(num_observations)
    cam = np.empty(ne, np.uint32)
    pt = np.empty(ne, np.uint32)
    obs = np.empty((ne, 2), np.float64)
    cams = np.empty((nc, 9), np.float64)
    pts = np.empty((np_, 3), np.float64)
    rc = _abi.lib().gb_synthetic_bal(nc, np_, ne, seed, camera_stride, zipf, cam.ctypes.data, pt.ctypes.data,
                                     obs.ctypes.data, cams.ctypes.data, pts.ctypes.data)
    if rc != _abi.GB_OK:
        raise ValueError("synthetic_bal: invalid shape (need observations >= points and degree <= cameras)")
    return BALProblem(cams, pts, cam, pt, obs)


def parse_bal_text(text: str) -> BALProblem:
    """bal/problem.hpp:46-55, src/bal_problem.cpp:81-115 (header, observations, cameras, points)."""
    tok = text.split()
    pos = 0

    def take(n):
        nonlocal pos
        if pos + n > len(tok):
            raise ValueError("truncated file")
        out = tok[pos:pos + n]
        pos += n
        return out

    nc, np_, ne = (int(v) for v in take(3))
    raw = np.array(take(4 * ne), dtype=object).reshape(ne, 4) if ne else np.zeros((0, 4), dtype=object)
    cam = raw[:, 0].astype(np.uint64)
    pt = raw[:, 1].astype(np.uint64)
    if ne and (cam.max() >= nc or pt.max() >= np_):
        raise ValueError("observation index out of range")
    obs = raw[:, 2:4].astype(np.float64)
    cams = np.array(take(9 * nc), dtype=np.float64).reshape(nc, 9)
    pts = np.array(take(3 * np_), dtype=np.float64).reshape(np_, 3)
    return BALProblem(cams, pts, cam.astype(np.uint32), pt.astype(np.uint32), obs.reshape(ne, 2))


def serialize_bal_text(p: BALProblem) -> str:
    """src/bal_problem.cpp:121-136 (%.17g round trip)."""
    lines = [f"{p.num_cameras} {p.num_points} {p.num_observations}"]
    for c, q, (x, y) in zip(p.camera_index, p.point_index, p.observations):
        lines.append(f"{int(c)} {int(q)} {x:.17g} {y:.17g}")
    lines.extend(f"{v:.17g}" for v in p.cameras.reshape(-1))
    lines.extend(f"{v:.17g}" for v in p.points.reshape(-1))
    return "\n".join(lines) + "\n"


# ---------------------------------------------------------------- the graph
class Backend:
    """A C ABI implementing include/gb_bal.h (the device library, or the
    reference compiled as the oracle with prefix 'ref_')."""

    def __init__(self, lib: ctypes.CDLL, prefix: str):
        self.lib = lib
        self.prefix = prefix

    def fn(self, name):
        return getattr(self.lib, self.prefix + name)

    def create(self, precision: int, mode: int, arg: int):
        return self.fn("create")(precision, mode, arg)

    def check(self, rc: int):
        if rc == _abi.GB_OK:
            return
        msg = self.fn("last_error")().decode()
        if rc == _abi.GB_ERR_INVALID_ARGUMENT:
            raise ValueError(msg)
        if rc == _abi.GB_ERR_OUT_OF_RANGE:
            raise IndexError(msg)
        if rc == _abi.GB_ERR_LOGIC:
            raise LogicError(msg)
        if rc == _abi.GB_ERR_RUNTIME:
            raise RuntimeError(msg)
        raise DeviceError(msg)


def device_backend() -> Backend:
    return Backend(_abi.lib(), "gb_")


class _PinnedBlock:
    """A gb_host_alloc block exposed to numpy; freed (returned to the
    library's cache) when the last array viewing it goes away."""

    def __init__(self, backend: "Backend", nbytes: int):
        self._free = backend.fn("host_free")
        self.ptr = backend.fn("host_alloc")(max(1, nbytes))
        self.__array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (self.ptr or 0, False),
                                    "version": 3}

    def __del__(self):
        if self.ptr:
            self._free(self.ptr)
            self.ptr = None


def _owned_array(src, dtype, backend: "Backend") -> np.ndarray:
    """A contiguous copy of src owned by the graph: page-locked memory from the
    device library when available (full-rate upload and write-back), else an
    ordinary numpy copy."""
    a = np.ascontiguousarray(src, dtype=dtype)
    if backend.prefix == "gb_" and a.nbytes:
        blk = _PinnedBlock(backend, a.nbytes)
        if blk.ptr:
            out = np.asarray(blk).view(a.dtype).reshape(a.shape)
            backend.fn("host_copy")(out.ctypes.data, a.ctypes.data, a.nbytes)
            return out
    return a.copy()


class BalGraph:
    """bal::BalGraph (adapter.hpp:82-100): owns the camera and point arrays
    (AoS, graph precision) that the solver refines IN PLACE."""

    def __init__(self, problem: BALProblem, precision: str = "fp64", diff_mode: str = "analytic",
                 huber_delta: Optional[float] = None, device: int = 0, backend: Optional[Backend] = None,
                 create_arg: Optional[int] = None):
        if precision not in PRECISIONS:
            raise ValueError(f"invalid precision pair: {precision}")
        if diff_mode not in MODES:
            raise ValueError(f"unknown differentiation mode: {diff_mode}")
        self.precision = precision
        self.diff_mode = diff_mode
        self.backend = backend or device_backend()
        self.FP, self.SP, self.A = dtypes(precision)
        self.num_observations = problem.num_observations
        self.cameras = _owned_array(problem.cameras, self.FP, self.backend)
        self.points = _owned_array(problem.points, self.FP, self.backend)
        self._cam_idx = np.ascontiguousarray(problem.camera_index, dtype=np.uint32)
        self._pt_idx = np.ascontiguousarray(problem.point_index, dtype=np.uint32)
        self._obs = np.ascontiguousarray(problem.observations, dtype=self.FP)
        h = self.backend.create(PRECISIONS[precision], MODES[diff_mode], device if create_arg is None else create_arg)
        if not h:
            self.backend.check(_abi.GB_ERR_NO_DEVICE if self.backend.prefix == "gb_" else _abi.GB_ERR_INVALID_ARGUMENT)
        self._h = h
        self._cam_fixed = None
        self._pt_fixed = None
        self._levels = None
        self._loss = (_abi.GB_LOSS_HUBER, float(huber_delta)) if huber_delta is not None else (_abi.GB_LOSS_DEFAULT, 1.0)
        self._bind()

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            self.backend.fn("destroy")(h)
            self._h = None

    def _bind(self):
        fn = self.backend.fn
        ptr = lambda a: None if a is None else a.ctypes.data  # noqa: E731
        self.backend.check(fn("set_cameras")(self._h, self.cameras.ctypes.data, self.cameras.shape[0],
                                             ptr(self._cam_fixed)))
        self.backend.check(fn("set_points")(self._h, self.points.ctypes.data, self.points.shape[0],
                                            ptr(self._pt_fixed)))
        self.backend.check(fn("set_observations")(self._h, self._cam_idx.shape[0], self._cam_idx.ctypes.data,
                                                  self._pt_idx.ctypes.data, self._obs.ctypes.data, ptr(self._levels),
                                                  self._loss[0], self._loss[1]))

    # -- structure edits
    def set_fixed(self, cameras=None, points=None):
        """VertexDescriptor::set_fixed for many vertices at once (boolean masks)."""
        if cameras is not None:
            self._cam_fixed = np.ascontiguousarray(cameras, dtype=np.uint8)
        if points is not None:
            self._pt_fixed = np.ascontiguousarray(points, dtype=np.uint8)
        self._bind()

    def set_levels(self, levels):
        """FactorDescriptor::set_level for every factor (uint8 per observation)."""
        self._levels = np.ascontiguousarray(levels, dtype=np.uint8)
        self._bind()

    # -- linear solver of the LM step
    def set_linear_solver(self, solver: str = "pcg"):
        """'pcg' (the reference's full-system PCG) or 'schur' (Schur complement
        onto the cameras, back-substituted points; device path only)."""
        if solver not in ("pcg", "schur"):
            raise ValueError(f"unknown linear solver: {solver}")
        self.backend.check(self.backend.fn("set_linear_solver")(self._h, 0 if solver == "pcg" else 1))

    # -- sharding (multi-GPU)
    def set_distributed(self, world: int, rank: int, kind: str = "nccl", uid: bytes = b""):
        """Shard this graph over `world` ranks (this handle is `rank`). kind
        'nccl': uid = nccl_unique_id() from rank 0; kind 'loopback': ranks are
        host threads of this process on one GPU, uid = an 8-byte group key;
        kind 'shm': one process per rank on this host (shared-memory
        collectives, any devices), uid = an 8-byte key equal on all ranks."""
        kinds = {"nccl": 0, "loopback": 1, "shm": 2}
        if kind not in kinds:
            raise ValueError(f"unknown reducer kind: {kind}")
        buf = ctypes.create_string_buffer(bytes(uid).ljust(128, b"\0"), 128)
        self.backend.check(self.backend.fn("set_distributed")(self._h, world, rank, kinds[kind], buf))
        self._bind()

    # -- objective
    def mse(self) -> float:
        out = ctypes.c_double()
        self.backend.check(self.backend.fn("mse")(self._h, ctypes.byref(out)))
        return out.value

    def total_error(self, level: int = 0) -> float:
        out = ctypes.c_double()
        self.backend.check(self.backend.fn("total_error")(self._h, level, ctypes.byref(out)))
        return out.value

    # -- LinearSystem surface (linear_system.hpp:44-216)
    def ls_linearize(self, level=0, clamp_min=1e-6, clamp_max=1e32, damping="after_scaling"):
        n = ctypes.c_int64()
        chi = ctypes.c_double()
        fin = ctypes.c_int32()
        # first call sizes N
        self.backend.check(self.backend.fn("ls_linearize")(self._h, level, clamp_min, clamp_max,
                                                           1 if damping == "before_scaling" else 0, ctypes.byref(chi),
                                                           ctypes.byref(n), None, None, None, None, ctypes.byref(fin)))
        N = n.value
        b, diag, cl, D = (np.zeros(N, self.FP) for _ in range(4))
        self.backend.check(self.backend.fn("ls_linearize")(self._h, level, clamp_min, clamp_max,
                                                           1 if damping == "before_scaling" else 0, ctypes.byref(chi),
                                                           ctypes.byref(n), b.ctypes.data, diag.ctypes.data,
                                                           cl.ctypes.data, D.ctypes.data, ctypes.byref(fin)))
        self._N = N
        return dict(chi2=chi.value, b=b, diag=diag, clamped=cl, scaling=D, finite=bool(fin.value), n=N)

    def ls_hvp(self, v, lam):
        v = _to_storage(v, self.SP)
        out = np.zeros(v.shape[0], self.A)
        self.backend.check(self.backend.fn("ls_hvp")(self._h, v.ctypes.data, out.ctypes.data, float(lam)))
        return out

    def ls_preconditioner(self, lam, nfree_cams, nfree_pts):
        blocks = np.zeros(81 * nfree_cams + 9 * nfree_pts, self.FP)
        fb = ctypes.c_int32()
        self.backend.check(self.backend.fn("ls_preconditioner")(self._h, float(lam), blocks.ctypes.data,
                                                                ctypes.byref(fb)))
        return blocks, fb.value

    def ls_solve_step(self, lam, pcg: PCGConfig):
        dx = np.zeros(self._N, self.FP)
        st = _abi.gb_pcg_stats()
        pred = ctypes.c_double()
        fin = ctypes.c_int32()
        c = pcg.to_c()
        self.backend.check(self.backend.fn("ls_solve_step")(self._h, float(lam), ctypes.byref(c), dx.ctypes.data,
                                                            ctypes.byref(st), ctypes.byref(pred), ctypes.byref(fin)))
        return dx, dict(iterations=st.iterations, final_relative_residual=st.final_relative_residual,
                        converged=bool(st.converged)), pred.value, bool(fin.value)

    def ls_jacobians(self, n_active):
        out = np.zeros((n_active, 24), self.SP)
        self.backend.check(self.backend.fn("ls_jacobians")(self._h, out.ctypes.data))
        return out

    def incidence(self, which: int):
        nseg, nit = ctypes.c_uint64(), ctypes.c_uint64()
        self.backend.check(self.backend.fn("incidence")(self._h, which, ctypes.byref(nseg), ctypes.byref(nit), None,
                                                        None, None, None))
        vos = np.zeros(nseg.value, np.uint64)
        off = np.zeros(nseg.value + 1, np.uint64)
        itf = np.zeros(nit.value, np.uint32)
        its = np.zeros(nit.value, np.uint16)
        self.backend.check(self.backend.fn("incidence")(self._h, which, ctypes.byref(nseg), ctypes.byref(nit),
                                                        vos.ctypes.data, off.ctypes.data, itf.ctypes.data,
                                                        its.ctypes.data))
        return vos, off, itf, its


def nccl_unique_id() -> bytes:
    """ncclGetUniqueId (128 bytes) through the library's runtime-loaded NCCL."""
    buf = ctypes.create_string_buffer(128)
    Backend(_abi.lib(), "gb_").check(_abi.lib().gb_nccl_unique_id(buf))
    return buf.raw


def shard_plan(problem: BALProblem, world: int):
    """Per-rank tile/point ranges, edge counts and point owners (host only)."""
    L = _abi.lib()
    tiles = np.zeros(2 * world, np.uint32)
    pts = np.zeros(2 * world, np.uint32)
    edges = np.zeros(world, np.uint64)
    owner = np.zeros(problem.num_points, np.uint32)
    cam = np.ascontiguousarray(problem.camera_index, np.uint32)
    pt = np.ascontiguousarray(problem.point_index, np.uint32)
    Backend(L, "gb_").check(L.gb_shard_plan(problem.num_cameras, problem.num_points, cam.shape[0], cam.ctypes.data,
                                            pt.ctypes.data, world, tiles.ctypes.data, pts.ctypes.data,
                                            edges.ctypes.data, owner.ctypes.data))
    return tiles.reshape(world, 2), pts.reshape(world, 2), edges, owner


def build_graph(problem: BALProblem, precision: str = "fp64", diff_mode: str = "analytic",
                huber_delta: Optional[float] = None, device: int = 0) -> BalGraph:
    """bal::build_graph<FP,SP> (adapter.hpp:106-143) on the B200 device path."""
    return BalGraph(problem, precision, diff_mode, huber_delta, device)


def _report(rep: _abi.gb_solve_report, recs) -> SolveReport:
    its = []
    for r in recs[: rep.iterations_run]:
        its.append(IterationRecord(r.iteration, r.chi2_before, r.chi2_after, r.lambda_, r.pcg_iterations,
                                   bool(r.pcg_converged), r.pcg_relative_residual, bool(r.low_quality_step),
                                   r.precond_fallback_blocks, bool(r.accepted), r.wall_seconds))
    m = rep.memory
    return SolveReport(its, rep.initial_chi2, rep.final_chi2, rep.accepted_steps,
                       _abi.TERMINATION_NAMES[rep.termination], rep.total_seconds, rep.free_dims, rep.residual_dims,
                       rep.active_factors,
                       dict(jacobian_bytes=m.jacobian_bytes, preconditioner_bytes=m.preconditioner_bytes,
                            workspace_bytes=m.workspace_bytes, graph_bytes=m.graph_bytes),
                       rep.setup_seconds, rep.h2d_bytes, rep.d2h_bytes)


def levenberg_marquardt(graph: BalGraph, config: Optional[LMConfig] = None) -> SolveReport:
    """levenberg_marquardt<FP,SP>(Graph&, const LMConfig&) (levenberg_marquardt.hpp:115-224).
    graph.cameras / graph.points are refined in place."""
    config = config or LMConfig()
    c = config.to_c()
    rep = _abi.gb_solve_report()
    n = max(1, config.max_iterations)
    recs = (_abi.gb_iteration_record * n)()
    graph.backend.check(graph.backend.fn("optimize")(graph._h, ctypes.byref(c), ctypes.byref(rep), recs, n))
    return _report(rep, recs)
