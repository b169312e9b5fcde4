"""The C++ facade (include/gopt_b200) compiles reference-style client code
unchanged and produces the same solve as the Python mirror and the reference."""
import os
import re
import subprocess

import pytest

from paper_2509_26581_b200 import bal

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


NLOHMANN = "/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty"


def build_client(tmp_path):
    exe = str(tmp_path / "facade_bal")
    json_inc = ["-I", NLOHMANN] if os.path.isdir(NLOHMANN) else []
    subprocess.check_call(["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include", "gopt_b200"), "-I",
                           os.path.join(ROOT, "include")] + json_inc +
                          [os.path.join(ROOT, "tests", "cpp", "facade_bal.cpp"),
                           "-L", os.path.join(ROOT, "paper_2509_26581_b200"), "-lgb_bal", "-o", exe])
    return exe


def test_facade_compiles(tmp_path):
    assert os.path.exists(build_client(tmp_path))


@pytest.mark.gpu
def test_facade_solve_matches(gpu, ref, tmp_path):
    exe = build_client(tmp_path)
    env = dict(os.environ, LD_LIBRARY_PATH=os.path.join(ROOT, "paper_2509_26581_b200"))
    out = subprocess.run([exe], capture_output=True, text=True, env=env, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    rows = {m.group(1): dict(kv.split("=") for kv in m.group(2).split())
            for m in re.finditer(r"^(\S+) (iterations=.*)$", out.stdout, re.M)}
    p = bal.synthetic_bal(49, 7776, 31843, seed=42)
    cfg = bal.LMConfig(max_iterations=50)
    cfg.pcg.max_iterations = 10
    r = ref.build_graph(p, "fp64", workers=4)
    rr = bal.levenberg_marquardt(r, cfg)
    fp64 = rows["fp64"]
    assert int(fp64["iterations"]) == len(rr.iterations)
    assert abs(float(fp64["final_chi2"]) - rr.final_chi2) <= 1e-6 * rr.final_chi2
    assert abs(float(fp64["mse1"]) - r.mse()) <= 1e-6 * r.mse()
    for name in ("fp32", "fp32-bf16"):
        assert abs(float(rows[name]["final_chi2"]) - rr.final_chi2) <= 1e-4 * rr.final_chi2
    # to_csv: 2 header comments + column line + one row per iteration
    rep = dict(kv.split("=") for kv in re.search(r"^fp64-report (.*)$", out.stdout, re.M).group(1).split())
    assert int(rep["csv_lines"]) == 3 + int(fp64["iterations"]) and int(rep["json_bytes"]) > 100
