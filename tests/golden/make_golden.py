"""Regenerates the golden fixtures from the compiled reference (oracle/_ref).

Run in the build container (where /root/reference exists and `make -C oracle`
has built oracle/_ref/libgopt_ref.so):

    python tests/golden/make_golden.py

Outputs (committed): tests/golden/tiny_fp64.npz, tests/golden/known_answers.json.
The tiny problem is synthetic_bal(8, 60, 300, seed=11); the reference runs
with the BAL parity config (tests/acceptance.cpp:69-80: 50 LM iterations,
PCG 10 @ 1e-6).
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import refbind  # noqa: E402
from paper_2509_26581_b200 import bal  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def main():
    p = bal.synthetic_bal(8, 60, 300, seed=11)
    cfg = bal.LMConfig(max_iterations=50)
    cfg.pcg.max_iterations = 10
    r = refbind.build_graph(p, "fp64", workers=1)
    lin = r.ls_linearize(0)
    v = np.random.default_rng(123).standard_normal(lin["n"])
    hv = r.ls_hvp(v, 0.25)
    blocks, fb = r.ls_preconditioner(1e-3, 8, 60)
    dx, st, pred, fin = r.ls_solve_step(1e-3, bal.PCGConfig(max_iterations=10))
    inc = [r.incidence(w) for w in (0, 1)]
    jac = r.ls_jacobians(300)
    rep = bal.levenberg_marquardt(r, cfg)
    tr = np.array([[i.chi2_before, i.chi2_after, i.lambda_, i.pcg_iterations, i.accepted] for i in rep.iterations])
    np.savez_compressed(
        os.path.join(OUT, "tiny_fp64.npz"), cameras=p.cameras, points=p.points, camera_index=p.camera_index,
        point_index=p.point_index, observations=p.observations, chi2=lin["chi2"], b=lin["b"], diag=lin["diag"],
        scaling=lin["scaling"], hvp_v=v, hvp_out=hv, precond=blocks, dx=dx, pred=pred, pcg_its=st["iterations"],
        jacobians=jac, cam_vos=inc[0][0], cam_off=inc[0][1], cam_items=inc[0][2], pt_vos=inc[1][0],
        pt_off=inc[1][1], pt_items=inc[1][2], trace=tr, final_cameras=r.cameras, final_points=r.points,
        final_chi2=rep.final_chi2, termination=rep.termination)
    ka = {}
    cam = [0, 0, 0, 0, 0, 0, 100.0, 0, 0]
    ka["project_origin"] = list(refbind.snavely_project(cam, [0, 0, -1]))
    ka["project_x1"] = list(refbind.snavely_project(cam, [1, 0, -1]))
    cam[7] = 0.1
    ka["project_k1"] = list(refbind.snavely_project(cam, [1, 0, -1]))
    ka["rotate_half_pi"] = list(refbind.rotate_angle_axis([0, 0, np.pi / 2], [1, 0, 0]))
    ka["nielsen"] = [refbind.update_damping(1.0, 2.0, False, 0.0), refbind.update_damping(3.0, 4.0, True, 1.0),
                     refbind.update_damping(3.0, 2.0, True, 0.5)]
    vals = [1.0, -2.5, 3.14159, 1e-30, 65504.0, 1.00390625, 1.01171875, float("inf"), -float("inf")]
    ka["bf16"] = [[v, refbind.bf16_round(v)] for v in vals]
    ka["bf16_nan"] = refbind.bf16_round(float("nan"))
    rng = np.random.default_rng(44)
    jc_cases = []
    for _ in range(5):
        c = np.concatenate([rng.normal(0, 0.4, 3), rng.normal(0, 1, 3), [rng.uniform(300, 1500)],
                            [rng.normal(0, 0.1)], [rng.normal(0, 0.01)]])
        x = rng.normal(0, 2, 3)
        jc, jp = refbind.snavely_jacobians(c, x)
        jc_cases.append(dict(camera=list(c), point=list(x), jc=jc.reshape(-1).tolist(), jp=jp.reshape(-1).tolist(),
                             pred=list(refbind.snavely_project(c, x))))
    ka["jacobian_cases"] = jc_cases
    with open(os.path.join(OUT, "known_answers.json"), "w") as f:
        json.dump(ka, f, indent=1)
    print("wrote golden fixtures:", rep.termination, len(rep.iterations), rep.final_chi2)


if __name__ == "__main__":
    main()
