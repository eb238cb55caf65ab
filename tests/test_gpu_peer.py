"""The multi-GPU MIN merge fused into the compose kernel over peer memory
(opsc_compose_argmin_peers + opsc_peer_barrier, dist.PeerMerge)."""

import os
import subprocess
import sys

import numpy as np
import pytest
import torch

from paper_2511_02248_b200 import _native, abi, device, dist as pdist, model, tables
from workloads import scenarios

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def _cfg5(n=48):
    prob = tables.pack_problem(*scenarios.scenario("cfg5"))
    grid = tables.pack_grid(prob, model.AutoscaleParams(slo=0.5), model.BruteForceBounds(**scenarios.GRIDS["cfg5"]))
    tw = scenarios.trace_windows("cfg5")
    idx = np.linspace(0, 1439, n).round().astype(int)
    return prob, grid, tables.window_arrays(tw["prefill_qps"][idx], tw["prefill_len"][idx], 0, 0.5)


def test_peer_atomics_reach_every_destination():
    """Two shards, each min-reducing into two destination buffers: both
    buffers end with the single-launch keys."""
    prob, grid, win = _cfg5()
    planner = device.DevicePlanner(prob, win, abi.MODE_ORACLE, grid=grid)
    planner.step()
    want = planner.key.clone()
    L, r = _native.load(), _native.ref
    import ctypes as C
    dst = [torch.full((win.n,), abi.KEY_INFEASIBLE, dtype=torch.int64, device="cuda") for _ in range(2)]
    ptrs = (C.c_void_p * 2)(*[t.data_ptr() for t in dst])
    s = torch.cuda.current_stream().cuda_stream
    for shard in range(3):
        _native.check(L.opsc_compose_argmin_peers(r(prob.table), r(grid), planner.win, planner.menu.data_ptr(),
                                                  shard, 3, ptrs, 2, s), "compose_peers")
    torch.cuda.synchronize()
    assert torch.equal(dst[0], want) and torch.equal(dst[1], want)


def test_peer_merge_single_rank_steps():
    """World size 1: PeerMerge's double-buffered steps equal the plain step."""
    prob, grid, win = _cfg5()
    a = device.DevicePlanner(prob, win, abi.MODE_ORACLE, grid=grid)
    a.step()
    want = a.decisions()
    b = device.DevicePlanner(prob, win, abi.MODE_ORACLE, grid=grid)
    merge = pdist.PeerMerge(win.n, "cuda")
    for _ in range(3):
        b.step(merge=merge)
        merge.check()
        got = b.decisions()
        for f in ("key", "cfg", "latency", "energy", "status"):
            assert getattr(got, f).tobytes() == getattr(want, f).tobytes(), f
    merge.close()


def test_peer_barrier_times_out_instead_of_hanging():
    """A barrier whose peer never arrives reports an error after the timeout."""
    import ctypes as C
    L = _native.load()
    flags = [torch.zeros(8, dtype=torch.int32, device="cuda") for _ in range(2)]
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    ptrs = (C.c_void_p * 2)(*[t.data_ptr() for t in flags])
    _native.check(L.opsc_peer_barrier(ptrs, 0, 2, 1, 200, err.data_ptr(),
                                      torch.cuda.current_stream().cuda_stream), "barrier")
    torch.cuda.synchronize()
    assert int(err.item()) == 1 and int(flags[1][0].item()) == 1  # arrival posted to the peer


def test_peer_merge_two_ranks_sharing_the_gpu():
    """Two processes (IPC on the same device; NVLink peers on a multi-GPU
    node use the same code) plan with the fused merge and agree with a
    single-rank plan on every step."""
    env = dict(os.environ, OPSC_DIST_BACKEND="gloo", PYTHONPATH=os.path.dirname(HERE))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29533", os.path.join(HERE, "peer_worker.py")]
    p = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, (p.stdout[-2000:], p.stderr[-3000:])
    assert p.stdout.count("ok") >= 2


def test_host_buffer_round_trip_single_rank():
    """dist.plan_windows_host_sharded (pinned host windows in, decisions out)
    equals the device-resident step, with and without the fused merge."""
    prob, grid, win = _cfg5(24)
    a = device.DevicePlanner(prob, win, abi.MODE_ORACLE, grid=grid)
    a.step()
    want = a.decisions()
    b = device.DevicePlanner(prob, tables.window_arrays(np.zeros(win.n), win.seq_len, 0, 0.5),
                             abi.MODE_ORACLE, grid=grid)
    merge = pdist.PeerMerge(win.n, "cuda")
    for m in (None, merge):
        out = tables.DecisionArrays(win.n, prob.n_ops)
        pdist.plan_windows_host_sharded(b, win, out, merge=m)
        for f in tables.DecisionArrays.FIELDS:
            assert getattr(out, f).tobytes() == getattr(want, f).tobytes(), (m, f)
    merge.close()


def _need_gpus(n):
    if torch.cuda.device_count() < n:
        pytest.skip(f"needs {n} GPUs, {torch.cuda.device_count()} visible")


def test_peer_merge_across_two_devices():
    """Two ranks on two DIFFERENT GPUs (NCCL group, CUDA-IPC handles opened on
    the peer device, NVLink atomics and the device barrier across the link):
    every rank's decisions equal a single-rank plan on every step."""
    _need_gpus(2)
    env = dict(os.environ, OPSC_DIST_BACKEND="nccl", PYTHONPATH=os.path.dirname(HERE))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29537", os.path.join(HERE, "peer_worker.py")]
    p = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, (p.stdout[-2000:], p.stderr[-3000:])
    assert p.stdout.count("ok") >= 2


def test_bench_two_gpus_self_spawned():
    """`bench.py --gpus 2` (no torchrun) spawns one rank per GPU and prints an
    n_gpus: 2 line whose decisions match the CPU oracle."""
    _need_gpus(2)
    import json
    repo = os.path.dirname(HERE)
    p = subprocess.run([sys.executable, os.path.join(repo, "bench.py"), "--gpus", "2", "--steps", "2",
                        "--warmup", "3", "--no-latency", "--no-cpu-baseline"],
                       capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, p.stderr[-3000:]
    line = json.loads(p.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 2 and line["parity_vs_oracle"] is True
    assert line["e2e"]["parity_vs_device_path"] is True


def test_bench_two_ranks_time_sharing_one_gpu():
    """The bench's N > 1 path end to end on the one GPU of this pool: two ranks
    under torchrun with the gloo process group (OPSC_DIST_BACKEND=gloo), the
    fused peer-memory merge between the two processes (CUDA IPC), sharded
    compose, e2e through dist.plan_windows_host_sharded: one n_gpus: 2 line
    whose decisions match the CPU oracle and the device path. Correctness of
    the N > 1 plumbing, not a scaling measurement."""
    import json
    repo = os.path.dirname(HERE)
    env = dict(os.environ, OPSC_DIST_BACKEND="gloo", PYTHONPATH=repo)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29541", os.path.join(repo, "bench.py"),
           "--gpus", "2", "--steps", "1", "--warmup", "3", "--no-latency", "--no-cpu-baseline"]
    p = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, (p.stdout[-2000:], p.stderr[-3000:])
    line = json.loads([x for x in p.stdout.strip().splitlines() if x.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["parity_vs_oracle"] is True
    assert line["e2e"]["parity_vs_device_path"] is True
    assert line["run"]["merge"].startswith("fused")
    assert line["order_certificate"]["order_sensitive_windows"] == 0
