"""bench.py at the driver's exact command line (--gpus 1 --steps 20
--warmup 5), on the Ladybug-shaped workload so it runs in seconds: exit code
0 and one complete JSON line (roofline, cpu_baseline, e2e, clocks, launches,
the timed window)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
def test_bench_driver_command_line(gpu):
    out = subprocess.run([sys.executable, "bench.py", "--gpus", "1", "--steps", "20", "--warmup", "5",
                          "--workload", "ladybug"], capture_output=True, text=True, cwd=ROOT, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["steps"] == 20 and d["warmup"] == 5 and d["n_gpus"] == 1
    assert d["value"] > 0 and d["unit"] == "ms/LM-iteration" and d["higher_is_better"] is False
    for k in ("roofline", "cpu_baseline", "e2e", "clocks", "gpu_launches", "window"):
        assert k in d, k
    assert d["roofline"]["frac"] > 0 and d["roofline"]["bound"] in ("hbm", "fp64", "fp32")
    assert d["cpu_baseline"]["value"] and d["cpu_baseline"]["kind"] == "reference"
    assert d["e2e"]["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] > 20
    assert d["window"]["accepted"] + d["window"]["rejected"] == 20
    assert d["solve"]["iterations"] == 25


@pytest.mark.gpu
def test_bench_reference_arm_same_window(gpu, ref):
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--gpus", "1", "--steps", "20",
                          "--warmup", "5", "--workload", "ladybug"], capture_output=True, text=True, cwd=ROOT,
                         timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    d = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][0])
    assert d["impl"] == "reference" and d["steps"] == 20 and d["warmup"] == 5
    assert d["window"]["accepted"] + d["window"]["rejected"] == 20
