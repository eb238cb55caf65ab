"""Compose-kernel edge cases on crafted menus, device keys against the CPU
oracle's literal enumeration on the SAME menu weights:

* sums landing within a few ulps of the SLO (ties at the 2^-40 grain,
  slo = 1.0 and non-power-of-two slos), which separates an exact mask from
  any high-word or threshold shortcut and checks the weight-sorted feasible-
  prefix count;
* slo = +inf with unstable (INF-weighted) entries: only all-finite candidates
  qualify, as in the reference's skip of non-finite weights
  (autoscaler.py:800-801);
* a menu with negative weights (the kernel's exact-scan path);
* chain (CHAIN kernel) and merge / fork DAGs (generic kernel), j menus from
  4 to 32 entries (every NJ specialisation) and > 32 (smem loop);
* menus too large for the shared-memory tile (the flat kernel), sharded.
"""

import zlib

import numpy as np
import pytest

from paper_2511_02248_b200 import abi, model, tables

pytestmark = pytest.mark.gpu

ULP40 = 2.0 ** -40


@pytest.fixture(scope="module")
def nat_loaded():
    from paper_2511_02248_b200 import _native
    _native.load()
    assert _native.device_count() >= 1, "no CUDA device"
    return _native


def _dag(n, shape):
    ids = [f"op{chr(97 + i)}" for i in range(n)]
    if shape == "chain":
        edges = [(ids[i], ids[i + 1]) for i in range(n - 1)]
    elif shape == "merge":
        edges = [(ids[i], ids[i + 1]) for i in range(n - 3)] + [(ids[n - 3], ids[n - 1]), (ids[n - 2], ids[n - 1])]
    else:  # fork: two sinks
        edges = [(ids[i], ids[i + 1]) for i in range(n - 2)] + [(ids[n - 3], ids[n - 1])]
    nodes = [{"id": i, "kind": "linear", "layer_count": 1, "profile_ref": "p" + i} for i in ids]
    prof = {"_link_bandwidth": 900e9}
    for i in ids:
        prof["p" + i] = {"prefill": {"c0": 1e-5, "c1": 1e-8}, "decode": {"c0": 1e-5, "c1": 1e-8},
                         "weight_mem": 1e8, "m1": 1e4, "v1": 1e4, "s0": 0.1, "s1": 1e-4}
    dag = {"nodes": nodes, "edges": [{"src": a, "dst": b, "volume_ref": "p" + a} for a, b in edges]}
    return tables.pack_problem(model.build_dag(dag), model.profiles_from_dict(prof))


def _menus(rng, prob, grid, slos, kind):
    """Menu weights whose candidate latencies crowd the SLO at the 2^-40 grain.
    Every path of the DAGs here visits n_path ops; each op's weight is
    slo/n_path plus a few 2^-40 steps, so sums are exact and tie the SLO."""
    n = prob.n_ops
    E = grid.menu_off[n]
    # per-entry cost P*R in the menu's (P, R, B) order; cheaper entries are
    # heavier (as on real menus), so the argmin sits in the SLO's tie band
    cost = np.concatenate([[p * r for p in (1, 2) for r in range(1, grid.r_max + 1) for _ in range(grid.b_max[v])]
                           for v in range(n)]).astype(np.float64)
    assert cost.size == E
    mw = np.empty((len(slos), E))
    for w, slo in enumerate(slos):
        base = (1.0 if not np.isfinite(slo) else slo) / (n if kind != "short" else n - 1)
        base = np.ldexp(np.round(np.ldexp(base, 40)), -40)  # on the 2^-40 grid
        mw[w] = base + (rng.integers(-3, 4, E) + 2.0 * (cost.mean() - cost)) * ULP40
        if kind == "inf":
            mw[w, rng.uniform(size=E) < 0.2] = np.inf
        if kind == "neg":
            mw[w, rng.uniform(size=E) < 0.1] *= -1.0
    return mw


@pytest.mark.parametrize("shape,n,r_max,b_max,kind", [
    ("chain", 6, 3, 2, "tie"), ("chain", 5, 2, 1, "tie"), ("chain", 5, 4, 1, "tie"),
    ("chain", 5, 3, 4, "tie"), ("chain", 4, 4, 4, "tie"), ("chain", 4, 6, 3, "tie"),
    ("chain", 6, 3, 2, "inf"), ("chain", 6, 3, 2, "neg"),
    ("merge", 6, 3, 2, "tie"), ("fork", 6, 3, 2, "tie"), ("fork", 6, 3, 2, "inf"), ("merge", 6, 3, 2, "neg"),
])
def test_compose_edges_vs_oracle(nat_loaded, orc, shape, n, r_max, b_max, kind):
    import torch

    from paper_2511_02248_b200 import _native as nat
    rng = np.random.default_rng(zlib.crc32(repr((shape, n, r_max, b_max, kind)).encode()))
    prob = _dag(n, shape)
    grid = tables.pack_grid(prob, model.AutoscaleParams(slo=1.0),
                            model.BruteForceBounds(r_max=r_max, b_max=b_max, parallelism=(1, 2)))
    slos = [1.0, 0.7, 0.3 + 1e-13, 2.5, 1.0, 0.9999999999999999]
    if kind == "inf":
        slos = [np.inf, np.inf, 1.0, np.inf]
    W = len(slos)
    win = tables.window_arrays(np.full(W, 10.0), np.full(W, 512), 0, 1.0)
    win.slo[:] = slos
    mw = _menus(rng, prob, grid, slos, kind if shape == "chain" else ("short" if kind == "tie" else kind))

    want = orc.compose(prob, grid, win, mw)
    dev = torch.device("cuda:0")
    t = {k: torch.from_numpy(np.ascontiguousarray(getattr(win, k))).to(dev)
         for k in ("qps", "seq_len", "phase", "slo", "eps")}
    dw = abi.OpscWindows()
    dw.n = W
    for k in t:
        setattr(dw, k, t[k].data_ptr())
    mwd = torch.from_numpy(mw).to(dev)
    key = torch.full((W,), abi.KEY_INFEASIBLE, dtype=torch.int64, device=dev)
    s = torch.cuda.current_stream().cuda_stream
    L = nat.load()
    nat.check(L.opsc_compose_argmin(nat.ref(prob.table), nat.ref(grid), dw, mwd.data_ptr(), 0, 1,
                                    key.data_ptr(), s), "compose")
    got = key.cpu().numpy()
    assert (got == want).all(), (shape, kind, got, want)
    if kind == "inf":
        assert (got != abi.KEY_INFEASIBLE).any()


def _device_compose(nat, prob, grid, win, mw, shard=0, n_shards=1):
    import torch
    dev = torch.device("cuda:0")
    t = {k: torch.from_numpy(np.ascontiguousarray(getattr(win, k))).to(dev)
         for k in ("qps", "seq_len", "phase", "slo", "eps")}
    dw = abi.OpscWindows()
    dw.n = win.n
    for k in t:
        setattr(dw, k, t[k].data_ptr())
    mwd = torch.from_numpy(np.ascontiguousarray(mw)).to(dev)
    key = torch.full((win.n,), abi.KEY_INFEASIBLE, dtype=torch.int64, device=dev)
    L = nat.load()
    nat.check(L.opsc_compose_argmin(nat.ref(prob.table), nat.ref(grid), dw, mwd.data_ptr(), shard, n_shards,
                                    key.data_ptr(), torch.cuda.current_stream().cuda_stream), "compose")
    return key.cpu().numpy()


@pytest.mark.parametrize("shape,r_max,b_max", [("chain", 512, 20), ("fork", 128, 10)])
def test_flat_kernel_large_menus(nat_loaded, orc, shape, r_max, b_max):
    """Two 20480-entry menus (past the shared-memory tile: the flat kernel)
    and three 2560-entry menus (the tile's shared-memory j loop)."""
    from paper_2511_02248_b200 import _native as nat
    n = 2 if shape == "chain" else 3
    rng = np.random.default_rng(r_max + b_max)
    prob = _dag(n, shape)
    grid = tables.pack_grid(prob, model.AutoscaleParams(slo=1.0),
                            model.BruteForceBounds(r_max=r_max, b_max=b_max, parallelism=(1, 2)))
    slos = [1.0, 0.7, np.inf, 0.3]
    W = len(slos)
    win = tables.window_arrays(np.full(W, 10.0), np.full(W, 512), 0, 1.0)
    win.slo[:] = slos
    mw = _menus(rng, prob, grid, slos, "inf" if shape == "chain" else "short")
    want = orc.compose(prob, grid, win, mw)
    got = _device_compose(nat, prob, grid, win, mw)
    assert (got == want).all(), (got, want)
    merged = np.minimum.reduce([_device_compose(nat, prob, grid, win, mw, sh, 3) for sh in range(3)])
    assert (merged == want).all()
    assert (got != abi.KEY_INFEASIBLE).any()


_SPLIT_ORACLE = {}


@pytest.mark.parametrize("cfg", ["cfg2", "cfg3"])
@pytest.mark.parametrize("il", [2, 3, 4, 5, 6])
def test_level_splits_vs_oracle(nat_loaded, orc, cfg, il, monkeypatch):
    """Every in-thread level count on the 10-op 70B path DAG (cfg2, MODE 2)
    and the 12-op two-source multimodal DAG (cfg3, generic MODE): il - 2
    middle levels run as the register odometer (0..4 of them), the rest are
    decoded per thread (OPSC_COMPOSE_IL is the compose_setup dev override)."""
    from paper_2511_02248_b200 import _native as nat
    from workloads import scenarios
    prob = tables.pack_problem(*scenarios.scenario(cfg))
    g = scenarios.GRIDS[cfg]
    grid = tables.pack_grid(prob, model.AutoscaleParams(slo=1.0), model.BruteForceBounds(**g))
    tw = scenarios.trace_windows(cfg)
    idx = np.arange(0, 60, 6) if cfg == "cfg2" else np.array([3, 17, 30, 45])
    win = tables.window_arrays(tw["prefill_qps"][idx], tw["prefill_len"][idx], 0, 1.0)
    # SLOs 1x..6x the scenario's, so feasible and infeasible windows mix
    win.slo[:] = np.linspace(1.0, 6.0, len(idx)) * scenarios.SLO[cfg]["prefill"]
    if cfg not in _SPLIT_ORACLE:  # the oracle's answer does not depend on the split
        mw, _ = orc.menus(prob, grid, win)
        _SPLIT_ORACLE[cfg] = (mw, orc.compose(prob, grid, win, mw))
    mw, want = _SPLIT_ORACLE[cfg]
    monkeypatch.setenv("OPSC_COMPOSE_IL", str(il))
    got = _device_compose(nat, prob, grid, win, mw)
    assert (got == want).all(), (il, got, want)
    assert (got != abi.KEY_INFEASIBLE).any()


@pytest.mark.parametrize("cfg", ["cfg2", "cfg3"])
@pytest.mark.parametrize("spc", [2, 3, 7, 16, 1000])
def test_slices_per_cta_vs_oracle(nat_loaded, orc, cfg, spc, monkeypatch):
    """A CTA running `spc` consecutive 256-thread slices of its window (one
    table setup, one running minimum across slices; a partial last CTA when
    spc does not divide the slice count; 1000 = one CTA per window) gives the
    oracle's key (OPSC_COMPOSE_SPC is the compose_setup dev override)."""
    from paper_2511_02248_b200 import _native as nat
    from workloads import scenarios
    prob = tables.pack_problem(*scenarios.scenario(cfg))
    g = scenarios.GRIDS[cfg]
    grid = tables.pack_grid(prob, model.AutoscaleParams(slo=1.0), model.BruteForceBounds(**g))
    tw = scenarios.trace_windows(cfg)
    idx = np.arange(0, 60, 6) if cfg == "cfg2" else np.array([3, 17, 30, 45])
    win = tables.window_arrays(tw["prefill_qps"][idx], tw["prefill_len"][idx], 0, 1.0)
    win.slo[:] = np.linspace(1.0, 6.0, len(idx)) * scenarios.SLO[cfg]["prefill"]
    if cfg not in _SPLIT_ORACLE:
        mw, _ = orc.menus(prob, grid, win)
        _SPLIT_ORACLE[cfg] = (mw, orc.compose(prob, grid, win, mw))
    mw, want = _SPLIT_ORACLE[cfg]
    monkeypatch.setenv("OPSC_COMPOSE_SPC", str(spc))
    got = _device_compose(nat, prob, grid, win, mw)
    assert (got == want).all(), (spc, got, want)
    assert (got != abi.KEY_INFEASIBLE).any()
    # with the outer index space sharded over 3 ranks (uneven slice counts)
    parts = [_device_compose(nat, prob, grid, win, mw, shard=r, n_shards=3) for r in range(3)]
    assert (np.minimum.reduce(parts) == want).all(), spc


def test_boundary_count_vs_numpy(nat_loaded, orc):
    """opsc_compose_boundary counts the candidates within `band` ulps of slo:
    checked against a numpy enumeration of the same crafted tie menus (chain
    DP = plain adds in topological order)."""
    import itertools

    import torch

    from paper_2511_02248_b200 import _native as nat
    rng = np.random.default_rng(5)
    prob = _dag(4, "chain")
    grid = tables.pack_grid(prob, model.AutoscaleParams(slo=1.0),
                            model.BruteForceBounds(r_max=3, b_max=2, parallelism=(1, 2)))
    slos = [1.0, 0.7, 0.3 + 1e-13]
    win = tables.window_arrays(np.full(3, 10.0), np.full(3, 512), 0, 1.0)
    win.slo[:] = slos
    mw = _menus(rng, prob, grid, slos, "tie")
    mw[:, ::7] = np.inf  # unstable entries never count
    dev = torch.device("cuda:0")
    t = {k: torch.from_numpy(np.ascontiguousarray(getattr(win, k))).to(dev)
         for k in ("qps", "seq_len", "phase", "slo", "eps")}
    dw = abi.OpscWindows()
    dw.n = 3
    for k in t:
        setattr(dw, k, t[k].data_ptr())
    mwd = torch.from_numpy(mw).to(dev)
    topo = [int(v) for v in prob.table.topo[:prob.n_ops]]
    off = [grid.menu_off[v] for v in range(prob.n_ops + 1)]
    for band in (0.0, 3.0, 40.0):
        cnt = torch.zeros(3, dtype=torch.int64, device=dev)
        nat.check(nat.load().opsc_compose_boundary(nat.ref(prob.table), nat.ref(grid), dw, mwd.data_ptr(), band,
                                                   cnt.data_ptr(), torch.cuda.current_stream().cuda_stream),
                  "boundary")
        got = cnt.cpu().numpy()
        for w, slo in enumerate(slos):
            ulp = np.nextafter(slo, np.inf) - slo
            want = 0
            for combo in itertools.product(*[range(off[v], off[v + 1]) for v in topo]):
                lat = 0.0
                for e in combo:
                    lat = lat + mw[w, e]
                want += bool(np.isfinite(lat) and abs(lat - slo) <= band * ulp)
            assert got[w] == want, (band, w, got[w], want)
    assert got.sum() > 0
