"""The sharded (multi-GPU) solve path on one device.

gpurun provides one GPU, so the K-rank path runs as K host threads of this
process on the same device with the in-process loopback reducer (rank-order
reductions, the same kernels, partial/allreduce/finalize sites and final point
gather as under NCCL). NCCL itself is exercised with a one-rank communicator
(collective code path, NCCL calls captured into the iteration CUDA graph).
"""
import threading

import numpy as np
import pytest

from paper_2509_26581_b200 import bal

pytestmark = pytest.mark.gpu

LADYBUG = (49, 7776, 31843)


def cfg(its=50):
    c = bal.LMConfig(max_iterations=its)
    c.pcg.max_iterations = 10
    return c


def solve_sharded(problem, world, precision="fp64", key=1234, its=50):
    graphs = [bal.build_graph(problem, precision) for _ in range(world)]
    for r, g in enumerate(graphs):
        g.set_distributed(world, r, "loopback", int(key).to_bytes(8, "little"))
    reps = [None] * world
    errs = []

    def run(r):
        try:
            reps[r] = bal.levenberg_marquardt(graphs[r], cfg(its))
        except Exception as e:  # surfaced below
            errs.append(e)

    th = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(600)
    assert not errs, errs
    return graphs, reps


@pytest.mark.parametrize("world", [2, 3])
def test_loopback_shards_match_single_gpu(gpu, world):
    p = bal.synthetic_bal(*LADYBUG, seed=42)
    g1 = bal.build_graph(p, "fp64")
    r1 = bal.levenberg_marquardt(g1, cfg())
    graphs, reps = solve_sharded(p, world, key=100 + world)
    for g, r in zip(graphs, reps):
        assert r.termination == r1.termination and len(r.iterations) == len(r1.iterations)
        assert abs(r.final_chi2 - r1.final_chi2) <= 1e-9 * r1.final_chi2
        assert np.linalg.norm(g.points - g1.points) <= 1e-7 * np.linalg.norm(g1.points)
        assert np.linalg.norm(g.cameras - g1.cameras) <= 1e-7 * np.linalg.norm(g1.cameras)
        assert r.memory == r1.memory and r.free_dims == r1.free_dims
    # every rank ends with the same bits (replicated cameras, gathered points)
    for g in graphs[1:]:
        assert np.array_equal(g.cameras.view(np.uint64), graphs[0].cameras.view(np.uint64))
        assert np.array_equal(g.points.view(np.uint64), graphs[0].points.view(np.uint64))


def test_loopback_shards_fixed_and_heavy(gpu, ref):
    p = bal.synthetic_bal(520, 30, 30 * 520, seed=7)  # heavy single-point tiles
    fixed_c = np.zeros(520, bool)
    fixed_c[:5] = True
    graphs = [bal.build_graph(p, "fp64") for _ in range(2)]
    for r, g in enumerate(graphs):
        g.set_fixed(cameras=fixed_c)
        g.set_distributed(2, r, "loopback", (777).to_bytes(8, "little"))
    reps = [None, None]
    th = [threading.Thread(target=lambda r=r: reps.__setitem__(r, bal.levenberg_marquardt(graphs[r], cfg(12))))
          for r in range(2)]
    [t.start() for t in th]
    [t.join(600) for t in th]
    rr = ref.build_graph(p, "fp64", workers=4)
    rr.set_fixed(cameras=fixed_c)
    rb = bal.levenberg_marquardt(rr, cfg(12))
    assert len(reps[0].iterations) == len(rb.iterations)
    assert abs(reps[0].final_chi2 - rb.final_chi2) <= 1e-6 * rb.final_chi2
    assert np.array_equal(graphs[0].cameras[:5].view(np.uint64), p.cameras[:5].view(np.uint64))


def test_nccl_single_rank_collective_path(gpu):
    p = bal.synthetic_bal(*LADYBUG, seed=42)
    g1 = bal.build_graph(p, "fp64")
    r1 = bal.levenberg_marquardt(g1, cfg())
    g = bal.build_graph(p, "fp64")
    g.set_distributed(1, 0, "nccl", bal.nccl_unique_id())
    r = bal.levenberg_marquardt(g, cfg())
    assert len(r.iterations) == len(r1.iterations)
    assert abs(r.final_chi2 - r1.final_chi2) <= 1e-12 * r1.final_chi2


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_device_activation_matches_host_shard(gpu, world):
    """Each rank activates only its own point-tile range on the device; every
    array equals the host activation sliced by shard() (activate.cpp)."""
    from paper_2509_26581_b200 import _abi

    for i, p in enumerate([bal.synthetic_bal(*LADYBUG, seed=42), bal.synthetic_bal(200, 5000, 25000, seed=4, zipf=1.1),
                           bal.synthetic_bal(520, 30, 30 * 520, seed=7)]):
        for r in range(world):
            g = bal.build_graph(p, "fp64")
            if i == 0:
                rng = np.random.default_rng(3)
                g.set_fixed(cameras=rng.random(p.num_cameras) < 0.1, points=rng.random(p.num_points) < 0.05)
                g.set_levels((rng.random(p.num_observations) < 0.05).astype(np.uint8))
            g.set_distributed(world, r, "loopback", int(9000 + 10 * i + world).to_bytes(8, "little"))
            g.backend.check(_abi.lib().gb_activation_selfcheck(g._h, 0))


def _shm_rank(rank, world, key, q):
    import os
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2509_26581_b200 import bal as b

    p = b.synthetic_bal(*LADYBUG, seed=42)
    g = b.build_graph(p, "fp64", device=0)
    g.set_distributed(world, rank, "shm", int(key).to_bytes(8, "little"))
    r = b.levenberg_marquardt(g, cfg())
    q.put((rank, r.termination, len(r.iterations), r.final_chi2, g.cameras.copy(), g.points.copy()))


@pytest.mark.parametrize("world", [2])
def test_shm_processes_match_single_gpu(gpu, world):
    """The sharded solve as separate PROCESSES (one per rank, all on cuda:0)
    exchanging through the shared-memory reducer: the same answer as the
    single-GPU solve, and identical bits on every rank."""
    import multiprocessing as mpc
    import os

    p = bal.synthetic_bal(*LADYBUG, seed=42)
    g1 = bal.build_graph(p, "fp64")
    r1 = bal.levenberg_marquardt(g1, cfg())
    ctx = mpc.get_context("spawn")
    q = ctx.Queue()
    key = 0xC0FFEE00 + os.getpid() % 4096
    procs = [ctx.Process(target=_shm_rank, args=(r, world, key, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = sorted((q.get(timeout=600) for _ in range(world)), key=lambda t: t[0])
    for pr in procs:
        pr.join(60)
        assert pr.exitcode == 0
    for rank, term, nit, chi, cams, pts in res:
        assert term == r1.termination and nit == len(r1.iterations)
        assert abs(chi - r1.final_chi2) <= 1e-9 * r1.final_chi2
        assert np.linalg.norm(pts - g1.points) <= 1e-7 * np.linalg.norm(g1.points)
        assert np.array_equal(cams.view(np.uint64), res[0][4].view(np.uint64))
        assert np.array_equal(pts.view(np.uint64), res[0][5].view(np.uint64))
