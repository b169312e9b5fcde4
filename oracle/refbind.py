"""TEST INFRASTRUCTURE ONLY — ctypes binding of the compiled reference
(oracle/_ref/libgopt_ref.so, built by oracle/Makefile from the unmodified
/root/reference/proj sources + the Eigen-subset shim).

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may use this
module, and only as the checker / CPU baseline. It exposes the same Python
surface as the device path (paper_2509_26581_b200.bal.BalGraph) with the
reference's Graph::set_workers (graph.hpp:50) as the extra knob.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from paper_2509_26581_b200 import _abi
from paper_2509_26581_b200.bal import Backend, BalGraph

HERE = os.path.dirname(os.path.abspath(__file__))
REF_LIB = os.path.join(HERE, "_ref", "libgopt_ref.so")

_REF = None


def available() -> bool:
    return os.path.exists(REF_LIB)


def lib() -> ctypes.CDLL:
    global _REF
    if _REF is None:
        if not available():
            raise ImportError(f"{REF_LIB} missing: run `make -C oracle` where /root/reference exists")
        L = _abi.declare(ctypes.CDLL(REF_LIB), "ref_")
        L.ref_snavely_project.argtypes = [ctypes.c_void_p] * 3
        L.ref_snavely_project.restype = None
        L.ref_rotate_angle_axis.argtypes = [ctypes.c_void_p] * 3
        L.ref_rotate_angle_axis.restype = None
        L.ref_snavely_jacobians.argtypes = [ctypes.c_void_p] * 4
        L.ref_snavely_jacobians.restype = None
        L.ref_update_damping.argtypes = [ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double),
                                         ctypes.c_int, ctypes.c_double]
        L.ref_update_damping.restype = None
        L.ref_bf16_round.argtypes = [ctypes.c_float]
        L.ref_bf16_round.restype = ctypes.c_uint16
        _REF = L
    return _REF


def backend() -> Backend:
    return Backend(lib(), "ref_")


def build_graph(problem, precision="fp64", diff_mode="analytic", huber_delta=None, workers=1) -> BalGraph:
    """bal::build_graph on the compiled reference; workers = Graph::set_workers."""
    return BalGraph(problem, precision, diff_mode, huber_delta, backend=backend(), create_arg=workers)


def snavely_project(camera, point):
    c = np.ascontiguousarray(camera, np.float64)
    p = np.ascontiguousarray(point, np.float64)
    out = np.zeros(2)
    lib().ref_snavely_project(c.ctypes.data, p.ctypes.data, out.ctypes.data)
    return out


def rotate_angle_axis(omega, x):
    w = np.ascontiguousarray(omega, np.float64)
    v = np.ascontiguousarray(x, np.float64)
    out = np.zeros(3)
    lib().ref_rotate_angle_axis(w.ctypes.data, v.ctypes.data, out.ctypes.data)
    return out


def snavely_jacobians(camera, point):
    c = np.ascontiguousarray(camera, np.float64)
    p = np.ascontiguousarray(point, np.float64)
    jc = np.zeros(18)
    jp = np.zeros(6)
    lib().ref_snavely_jacobians(c.ctypes.data, p.ctypes.data, jc.ctypes.data, jp.ctypes.data)
    return jc.reshape(2, 9), jp.reshape(2, 3)


def update_damping(lam, nu, accepted, gain):
    l_, n_ = ctypes.c_double(lam), ctypes.c_double(nu)
    lib().ref_update_damping(ctypes.byref(l_), ctypes.byref(n_), int(accepted), float(gain))
    return l_.value, n_.value


def bf16_round(f: float) -> int:
    return int(lib().ref_bf16_round(float(f)))
