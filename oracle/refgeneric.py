"""TEST INFRASTRUCTURE ONLY: ctypes binding of oracle/_ref/libgopt_ref_generic.so,
the reference's generic CPU engine on the host-device models
(oracle/ref_generic.cpp). Same call surface as paper_2509_26581_b200.generic."""
import ctypes
import os

from paper_2509_26581_b200 import generic

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_ref", "libgopt_ref_generic.so")
_LIB = None


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _LIB
    if _LIB is None:
        _LIB = generic._declare(ctypes.CDLL(LIB_PATH), "refg_")
    return _LIB


def solve_circle(problem, precision="fp64", config=None, workers=1):
    return generic.solve_circle(problem, precision, config, lib=lib(), prefix="refg_", extra=workers)


def solve_vi(problem, precision="fp64", config=None, workers=1):
    return generic.solve_vi(problem, precision, config, lib=lib(), prefix="refg_", extra=workers)
