"""CPU checks of bench.py's plumbing: the --gpus N launcher decisions, the
torchrun command it spawns, a real 2-rank torchrun launch of the reference arm
(rank 0 alone works, rank 1 exits 0), and the provenance of the bench input:
the standalone writer gb_gen_bal produces exactly gb_synthetic_bal's problem,
and its %.17g BAL text reads back bit-identically through the reference's own
parser (src/bal_problem.cpp:81-136)."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def args(**kw):
    a = bench.parse_args([])
    for k, v in kw.items():
        setattr(a, k, v)
    return a


def test_resolve_world_single():
    assert bench.resolve_world(args(gpus=1), {}, 0) == "run"


def test_resolve_world_spawns_n_ranks():
    assert bench.resolve_world(args(gpus=8), {}, 8) == "spawn"


def test_resolve_world_fails_loudly_with_too_few_gpus():
    with pytest.raises(SystemExit, match="only 1 CUDA device"):
        bench.resolve_world(args(gpus=2), {}, 1)


def test_resolve_world_rejects_mismatched_torchrun_env():
    with pytest.raises(SystemExit, match="WORLD_SIZE=4"):
        bench.resolve_world(args(gpus=8), {"WORLD_SIZE": "4"}, 8)
    assert bench.resolve_world(args(gpus=4), {"WORLD_SIZE": "4"}, 0) == "run"


def test_reference_arm_never_spawns():
    assert bench.resolve_world(args(gpus=8, impl="reference"), {}, 0) == "run"


def test_launch_command():
    cmd = bench.launch_command(["--gpus", "2", "--steps", "20"], 2, 29555)
    assert cmd[:3] == [sys.executable, "-m", "torch.distributed.run"]
    assert "--nproc-per-node=2" in cmd and "127.0.0.1" in cmd and "--master-port=29555" in cmd
    assert cmd[-4:] == ["--gpus", "2", "--steps", "20"]
    assert cmd[cmd.index("--master-port=29555") + 1].endswith("bench.py")


def test_warmup_floor():
    assert bench.parse_args(["--warmup", "1"]).warmup == 3


def test_host_info():
    h = bench.host_info()
    assert h["os_cpu_count"] >= 1


def test_generator_matches_library():
    from paper_2509_26581_b200 import bal

    a = bench.load_problem(9, 200, 1100, seed=5)
    b = bal.synthetic_bal(9, 200, 1100, seed=5)
    for x, y in zip((a.cameras, a.points, a.camera_index, a.point_index, a.observations),
                    (b.cameras, b.points, b.camera_index, b.point_index, b.observations)):
        assert x.dtype == y.dtype and np.array_equal(x, y)


def test_generator_text_reads_back_through_reference_parser(tmp_path, ref):
    import ctypes

    path = tmp_path / "p.txt"
    with open(path, "wb") as f:
        subprocess.run([bench.GEN, "9", "200", "1100", "--seed", "5", "--text"], check=True, stdout=f)
    L = ref.lib()
    fn = L.ref_parse_bal_file
    fn.restype = ctypes.c_int
    fn.argtypes = [ctypes.c_char_p] + [ctypes.c_void_p] * 6
    shape = np.zeros(3, np.uint64)
    assert fn(str(path).encode(), shape.ctypes.data, None, None, None, None, None) == 0
    nc, np_, ne = (int(v) for v in shape)
    cam, pt = np.zeros(ne, np.uint32), np.zeros(ne, np.uint32)
    obs, cams, pts = np.zeros((ne, 2)), np.zeros((nc, 9)), np.zeros((np_, 3))
    assert fn(str(path).encode(), shape.ctypes.data, cam.ctypes.data, pt.ctypes.data, obs.ctypes.data,
              cams.ctypes.data, pts.ctypes.data) == 0
    b = bench.load_problem(9, 200, 1100, seed=5)
    assert np.array_equal(cam, b.camera_index) and np.array_equal(pt, b.point_index)
    assert np.array_equal(obs.view(np.uint64), b.observations.view(np.uint64))
    assert np.array_equal(cams.view(np.uint64), b.cameras.view(np.uint64))
    assert np.array_equal(pts.view(np.uint64), b.points.view(np.uint64))


def test_torchrun_two_ranks_reference_arm(ref):
    """A real 2-rank torchrun launch (127.0.0.1): rank 0 prints the reference
    line on the requested window, rank 1 exits 0 without work, and the
    reference process never loads the product library."""
    env = dict(os.environ, OMP_NUM_THREADS="1")
    cmd = bench.launch_command(["--impl", "reference", "--gpus", "2", "--workload", "ladybug", "--steps", "4",
                                "--warmup", "3"], 2, bench.free_port())
    out = subprocess.run(cmd, capture_output=True, text=True, env=env, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["steps"] == 4 and d["warmup"] == 3 and d["n_gpus"] == 2
    assert d["window"]["accepted"] + d["window"]["rejected"] == 4
    assert d["cpu_baseline"]["kind"] == "reference" and d["e2e"]["h2d_bytes_per_step"] == 0


def test_reference_arm_loads_only_oracle_library(ref):
    code = (
        "import sys, bench, os\n"
        "sys.argv = ['bench.py', '--impl', 'reference', '--workload', 'ladybug', '--steps', '3', '--warmup', '3']\n"
        "bench.main()\n"
        "maps = open('/proc/self/maps').read()\n"
        "print('PRODUCT_LOADED' if 'libgb_bal.so' in maps else 'PRODUCT_NOT_LOADED')\n")
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, cwd=ROOT, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    assert "PRODUCT_NOT_LOADED" in out.stdout
