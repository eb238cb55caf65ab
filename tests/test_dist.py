"""Multi-rank path on CPU (gloo, world_size 2): candidate-range shards +
MIN all-reduce of packed keys reproduce the single-process decision."""

import os
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2511_02248_b200 import abi, model, tables
from workloads import scenarios


def _inputs(cfg, phase, idx):
    prob = tables.pack_problem(*scenarios.scenario(cfg))
    g = scenarios.GRIDS[cfg]
    grid = tables.pack_grid(prob, model.AutoscaleParams(slo=1.0), model.BruteForceBounds(**g))
    tw = scenarios.trace_windows(cfg)
    win = tables.window_arrays(tw[phase + "_qps"][idx], tw[phase + "_len"][idx],
                               tables.PHASE_INDEX[phase], scenarios.SLO[cfg][phase])
    return prob, grid, win


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as orc
        from paper_2511_02248_b200 import dist as pdist
        res = {}
        for cfg, phase in (("cfg3s", "prefill"), ("cfg1", "decode"), ("cfg3s", "decode")):
            prob, grid, win = _inputs(cfg, phase, np.arange(0, 60, 6) if cfg == "cfg3s" else np.array([0]))
            mw, _ = orc.menus(prob, grid, win, n_threads=2)
            local = orc.compose(prob, grid, win, mw, shard=rank, n_shards=world, n_threads=2)
            keys = torch.from_numpy(local.copy())
            pdist.merge_keys(keys)
            res[(cfg, phase)] = keys.numpy().tolist()
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_min_allreduce_equals_single(world):
    from oracle import oracle as orc
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for (cfg, phase), keys in got[0].items():
        prob, grid, win = _inputs(cfg, phase, np.arange(0, 60, 6) if cfg == "cfg3s" else np.array([0]))
        mw, _ = orc.menus(prob, grid, win)
        single = orc.compose(prob, grid, win, mw)
        assert keys == single.tolist(), (cfg, phase)
        assert got[1][(cfg, phase)] == keys  # every rank holds the global decision
        assert any(k != abi.KEY_INFEASIBLE for k in keys) or cfg == "cfg3s"


def test_shard_ranges_cover_space(orc):
    """Shards of the oracle enumeration partition the space: min over any
    shard count equals the unsharded key."""
    prob, grid, win = _inputs("cfg3s", "prefill", np.arange(0, 60, 5))
    mw, _ = orc.menus(prob, grid, win)
    base = orc.compose(prob, grid, win, mw)
    for n in (2, 3, 5, 8):
        merged = np.full(win.n, abi.KEY_INFEASIBLE, dtype=np.int64)
        for s in range(n):
            merged = np.minimum(merged, orc.compose(prob, grid, win, mw, shard=s, n_shards=n))
        assert (merged == base).all()


def test_bench_refuses_more_gpus_than_visible():
    """`bench.py --gpus N` outside torchrun spawns N ranks itself, and fails
    loudly (exit 2) rather than printing an n_gpus: 1 line when fewer than N
    devices are visible (here: none)."""
    import subprocess
    import torch
    if torch.cuda.device_count() >= 2:
        pytest.skip("multi-GPU host")
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    p = subprocess.run([sys.executable, os.path.join(repo, "bench.py"), "--gpus", "2"],
                       capture_output=True, text=True, timeout=300)
    assert p.returncode == 2 and p.stdout == "", (p.returncode, p.stdout, p.stderr)
    assert "needs 2 CUDA devices" in p.stderr
    env = dict(os.environ, WORLD_SIZE="3", RANK="0", LOCAL_RANK="0")
    p = subprocess.run([sys.executable, os.path.join(repo, "bench.py"), "--gpus", "2"],
                       capture_output=True, text=True, timeout=300, env=env)
    assert p.returncode == 2 and "WORLD_SIZE=3" in p.stderr
