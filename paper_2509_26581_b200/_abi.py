"""ctypes mirror of include/gb_bal.h (structs, constants, library loading).

The product library is the in-tree ``libgb_bal.so`` built for sm_100a by
``__graft_entry__.build()`` (or ``make -C paper_2509_26581_b200/csrc``). There
is no CPU fallback: if the library is missing, importing the solver fails
loudly.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_double, c_int, c_int32, c_int64, c_uint8, c_uint16, c_uint32, c_uint64, c_void_p

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libgb_bal.so")

# status codes
GB_OK = 0
GB_ERR_INVALID_ARGUMENT = 1
GB_ERR_OUT_OF_RANGE = 2
GB_ERR_LOGIC = 3
GB_ERR_RUNTIME = 4
GB_ERR_CUDA = 5
GB_ERR_NO_DEVICE = 6

# precision pairs (src/experiment.cpp:153-157)
GB_FP64, GB_FP32, GB_FP32_BF16 = 0, 1, 2
# DifferentiationMode (factor_descriptor.hpp:23)
GB_ANALYTIC, GB_AUTO, GB_DYNAMIC = 0, 1, 2
GB_LOSS_DEFAULT, GB_LOSS_HUBER = 0, 1
GB_DAMPING_AFTER_SCALING, GB_DAMPING_BEFORE_SCALING = 0, 1

TERMINATION_NAMES = [
    "max_iterations",
    "tolerance_reached",
    "gradient_small",
    "damping_overflow",
    "non_finite_linearization",
    "no_free_parameters",
]


class gb_pcg_config(ctypes.Structure):
    _fields_ = [("max_iterations", c_int32), ("tolerance", c_double), ("rejection_ratio", c_double),
                ("normalize_rhs", c_int32)]


class gb_pcg_stats(ctypes.Structure):
    _fields_ = [("iterations", c_int32), ("final_relative_residual", c_double), ("converged", c_int32)]


class gb_lm_config(ctypes.Structure):
    _fields_ = [
        ("max_iterations", c_int32),
        ("tolerance", c_double),
        ("level", c_int32),
        ("tau", c_double),
        ("pcg", gb_pcg_config),
        ("clamp_min", c_double),
        ("clamp_max", c_double),
        ("damping", c_int32),
        ("use_rejection_guard", c_int32),
        ("refresh_on_reject", c_int32),
        ("lambda_max", c_double),
        ("gradient_tolerance", c_double),
    ]


class gb_iteration_record(ctypes.Structure):
    _fields_ = [
        ("iteration", c_int32),
        ("chi2_before", c_double),
        ("chi2_after", c_double),
        ("lambda_", c_double),
        ("pcg_iterations", c_int32),
        ("pcg_converged", c_int32),
        ("pcg_relative_residual", c_double),
        ("low_quality_step", c_int32),
        ("precond_fallback_blocks", c_int32),
        ("accepted", c_int32),
        ("wall_seconds", c_double),
    ]


class gb_memory_account(ctypes.Structure):
    _fields_ = [("jacobian_bytes", c_uint64), ("preconditioner_bytes", c_uint64), ("workspace_bytes", c_uint64),
                ("graph_bytes", c_uint64)]


class gb_solve_report(ctypes.Structure):
    _fields_ = [
        ("initial_chi2", c_double),
        ("final_chi2", c_double),
        ("accepted_steps", c_int32),
        ("termination", c_int32),
        ("total_seconds", c_double),
        ("free_dims", c_int64),
        ("residual_dims", c_int64),
        ("active_factors", c_uint64),
        ("memory", gb_memory_account),
        ("iterations_run", c_int32),
        ("setup_seconds", c_double),
        ("h2d_bytes", c_double),
        ("d2h_bytes", c_double),
    ]


# every symbol include/gb_bal.h declares (the CPU suite checks the export table)
EXPORTED = [
    "gb_default_config", "gb_last_error", "gb_device_count", "gb_create", "gb_destroy", "gb_set_cameras",
    "gb_set_points", "gb_set_observations", "gb_set_differentiation_mode", "gb_optimize", "gb_mse",
    "gb_total_error", "gb_ls_linearize", "gb_ls_hvp", "gb_ls_preconditioner", "gb_ls_solve_step",
    "gb_ls_jacobians", "gb_incidence", "gb_synthetic_bal", "gb_begin", "gb_step", "gb_end", "gb_stream",
    "gb_time_hvp", "gb_hvp_bytes", "gb_hvp_info", "gb_fma_peak", "gb_iteration_kernels", "gb_host_alloc", "gb_host_free", "gb_host_copy", "gb_nccl_unique_id", "gb_set_distributed", "gb_shm_allreduce_selftest", "gb_shard_plan", "gb_activation_selfcheck",
    "gb_set_linear_solver", "gb_report_json", "gb_report_csv",
    "gbg_last_error", "gbg_circle_solve", "gbg_vi_solve",  # generic path, include/gb_generic.h
]


def declare(lib: ctypes.CDLL, prefix: str = "gb_") -> ctypes.CDLL:
    """Attach argtypes/restypes for the gb_ (or ref_) C ABI."""
    P = prefix
    vp = c_void_p

    def f(name, res, *args):
        fn = getattr(lib, P + name)
        fn.restype = res
        fn.argtypes = list(args)

    f("last_error", c_char_p)
    f("destroy", None, vp)
    f("set_cameras", c_int, vp, vp, c_uint64, vp)
    f("set_points", c_int, vp, vp, c_uint64, vp)
    f("set_observations", c_int, vp, c_uint64, vp, vp, vp, vp, c_int, c_double)
    f("optimize", c_int, vp, POINTER(gb_lm_config), POINTER(gb_solve_report), vp, c_int32)
    f("mse", c_int, vp, POINTER(c_double))
    f("total_error", c_int, vp, c_int, POINTER(c_double))
    f("ls_linearize", c_int, vp, c_int, c_double, c_double, c_int, POINTER(c_double), POINTER(c_int64), vp, vp, vp,
      vp, POINTER(c_int32))
    f("ls_hvp", c_int, vp, vp, vp, c_double)
    f("ls_preconditioner", c_int, vp, c_double, vp, POINTER(c_int32))
    f("ls_solve_step", c_int, vp, c_double, POINTER(gb_pcg_config), vp, POINTER(gb_pcg_stats), POINTER(c_double),
      POINTER(c_int32))
    f("ls_jacobians", c_int, vp, vp)
    f("incidence", c_int, vp, c_int, POINTER(c_uint64), POINTER(c_uint64), vp, vp, vp, vp)
    if prefix == "gb_":
        f("default_config", None, POINTER(gb_lm_config))
        f("device_count", c_int)
        f("create", vp, c_int, c_int, c_int)
        f("set_differentiation_mode", c_int, vp, c_int)
        f("synthetic_bal", c_int, c_uint64, c_uint64, c_uint64, c_uint64, c_uint64, c_double, vp, vp, vp, vp, vp)
        f("begin", c_int, vp, POINTER(gb_lm_config), POINTER(gb_solve_report))
        f("step", c_int, vp, c_int32)
        f("end", c_int, vp, POINTER(gb_solve_report), vp, c_int32)
        f("stream", vp, vp)
        f("time_hvp", c_int, vp, c_int32, POINTER(c_double), POINTER(c_double))
        f("hvp_bytes", c_int, vp, POINTER(c_double), POINTER(c_double))
        f("hvp_info", c_int, vp, POINTER(c_int32), POINTER(c_double), POINTER(c_double), POINTER(c_double))
        f("fma_peak", c_int, c_int32, c_int32, POINTER(c_double))
        f("iteration_kernels", c_int, vp, POINTER(c_int32))
        f("host_alloc", vp, c_uint64)
        f("host_free", None, vp)
        f("host_copy", None, vp, vp, c_uint64)
        f("nccl_unique_id", c_int, vp)
        f("activation_selfcheck", c_int, vp, c_int)
        f("set_linear_solver", c_int, vp, c_int)
        f("set_distributed", c_int, vp, c_int, c_int, c_int, vp)
        f("report_json", c_int, POINTER(gb_solve_report), vp, c_int32, vp, c_uint64, POINTER(c_uint64))
        f("report_csv", c_int, POINTER(gb_solve_report), vp, c_int32, vp, c_uint64, POINTER(c_uint64))
        f("shm_allreduce_selftest", c_int, c_int, c_int, c_uint64, vp, c_uint64, c_int, vp, c_uint64)
        f("shard_plan", c_int, c_uint64, c_uint64, c_uint64, vp, vp, c_int, vp, vp, vp, vp)
    else:
        f("create", vp, c_int, c_int, c_int)
        f("set_workers", c_int, vp, c_int)
    return lib


_LIB = None


def lib() -> ctypes.CDLL:
    """The product library; raises (never falls back) when it is missing."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                "(the B200 solver has no CPU fallback)")
        _LIB = declare(ctypes.CDLL(LIB_PATH), "gb_")
    return _LIB
