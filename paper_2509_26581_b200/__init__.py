"""B200-native Levenberg–Marquardt bundle adjustment (the LM inner loop of
arXiv 2509.26581, reference `gopt`), behind the reference's API.

The solver is ``libgb_bal.so`` (hand-written sm_100a CUDA + a C ABI,
include/gb_bal.h); this package is the thin host-side mirror used by tests,
the benchmark and Python callers. C++ callers use include/gopt_b200/.
"""
from .bal import (  # noqa: F401
    BALProblem,
    BalGraph,
    IterationRecord,
    LMConfig,
    LogicError,
    PCGConfig,
    SolveReport,
    build_graph,
    levenberg_marquardt,
    parse_bal_text,
    serialize_bal_text,
    synthetic_bal,
)

__all__ = [
    "BALProblem", "BalGraph", "IterationRecord", "LMConfig", "LogicError", "PCGConfig", "SolveReport",
    "build_graph", "levenberg_marquardt", "parse_bal_text", "serialize_bal_text", "synthetic_bal",
]
