"""Evidence (reference only, CPU): at tolerance 1e-6 the REFERENCE's own fp32 /
fp32-bf16 LM iteration count is decided by rounding noise. The same Ladybug-
shaped problem with its observations merely listed in a different order (an
equivalent problem: the same factors, a different summation order in the
reference's sequential chi^2 and CSR accumulation) converges after a
different number of iterations, while fp64 and tolerance 1e-4 do not move.

  python tools/ref_order_noise.py > profiles/r02_ref_order_noise.md
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import refbind  # noqa: E402
from paper_2509_26581_b200 import bal  # noqa: E402


def permuted(p, seed):
    perm = np.random.default_rng(seed).permutation(p.num_observations)
    return bal.BALProblem(p.cameras, p.points, p.camera_index[perm], p.point_index[perm], p.observations[perm])


def run(prob, prec, tol, workers=8):
    c = bal.LMConfig(max_iterations=50, tolerance=tol)
    c.pcg.max_iterations = 10
    rep = bal.levenberg_marquardt(refbind.build_graph(prob, prec, workers=workers), c)
    return len(rep.iterations), rep.termination, rep.final_chi2


def main():
    p = bal.synthetic_bal(49, 7776, 31843, seed=42)
    print("# The reference's own LM iteration count under observation-order permutations\n")
    print("Ladybug-49-shaped synthetic BA (seed 42), the compiled reference (oracle/_ref), 50 LM iterations, "
          "PCG 10 @ 1e-6. Column 'as given' is the generator's point-grouped order; perm k is "
          "`np.random.default_rng(k).permutation` of the observations (same factors).\n")
    print("| precision | tolerance | as given | perm 0 | perm 1 | perm 2 | perm 3 |")
    print("|---|---|---|---|---|---|---|")
    for prec in ["fp64", "fp32", "fp32-bf16"]:
        for tol in [1e-6, 1e-4]:
            out = [run(p, prec, tol)] + [run(permuted(p, s), prec, tol) for s in range(4)]
            cells = [f"{n} ({t.split('_')[0]}, {c:.9g})" for n, t, c in out]
            print(f"| {prec} | {tol:g} | " + " | ".join(cells) + " |")


if __name__ == "__main__":
    main()
