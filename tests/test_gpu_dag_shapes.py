"""Exhaustive compose on non-chain DAGs at scale (the generic, non-CHAIN
kernel path: merges, forks, multi-sink) and on the 12-op multimodal DAG --
GPU decisions and every plan field against the CPU oracle."""

import numpy as np
import pytest

from paper_2511_02248_b200 import abi, model, tables
from workloads import scenarios

pytestmark = pytest.mark.gpu


def _random_dag(rng, n, shape):
    ids = [f"op{chr(97 + i)}" for i in range(n)]
    if shape == "merge":      # last node merges two branches
        edges = [(ids[i], ids[i + 1]) for i in range(n - 3)] + [(ids[n - 3], ids[n - 1]), (ids[n - 2], ids[n - 1])]
    elif shape == "fork":     # two sinks
        edges = [(ids[i], ids[i + 1]) for i in range(n - 2)] + [(ids[n - 3], ids[n - 1])]
    elif shape == "early_sink":  # a->b->c (sink c above the in-thread levels), b->d->...->last
        edges = [(ids[0], ids[1]), (ids[1], ids[2]), (ids[1], ids[3])] + [(ids[i], ids[i + 1]) for i in range(3, n - 1)]
    elif shape == "two_source":  # a->b->c and d->c, then a chain (merge above the in-thread levels)
        edges = [(ids[0], ids[1]), (ids[1], ids[2]), (ids[3], ids[2])] + [(ids[2], ids[4])] + \
                [(ids[i], ids[i + 1]) for i in range(4, n - 1)]
    else:                     # random DAG
        edges = [(ids[i], ids[j]) for j in range(1, n) for i in range(j) if rng.uniform() < 0.35]
    nodes = [{"id": i, "kind": "linear", "layer_count": int(rng.choice([1, 8, 32])), "profile_ref": "p" + i}
             for i in ids]
    prof = {"_link_bandwidth": 900e9}
    for i in ids:
        c0, c1 = float(rng.uniform(2e-6, 3e-5)), float(10 ** rng.uniform(-9, -6.8))
        prof["p" + i] = {"prefill": {"c0": c0, "c1": c1}, "decode": {"c0": c0, "c1": c1},
                         "weight_mem": 1e8, "m1": 1e4, "v1": float(rng.uniform(4e3, 4e4)),
                         "s0": 0.1, "s1": 1e-4}
    dag = {"nodes": nodes, "edges": [{"src": a, "dst": b, "volume_ref": "p" + a} for a, b in edges]}
    return model.build_dag(dag), model.profiles_from_dict(prof)


@pytest.mark.parametrize("shape,n", [("merge", 7), ("fork", 7), ("random", 7), ("random", 8),
                                     ("early_sink", 7), ("early_sink", 8), ("two_source", 7), ("two_source", 8)])
def test_generic_dag_exhaustive_vs_oracle(nat_loaded, orc, shape, n):
    from paper_2511_02248_b200 import _native
    rng = np.random.default_rng(n * 7 + len(shape))
    dag, prof = _random_dag(rng, n, shape)
    prob = tables.pack_problem(dag, prof)
    grid = tables.pack_grid(prob, model.AutoscaleParams(slo=1.0),
                            model.BruteForceBounds(r_max=3, b_max=2, parallelism=(1, 2)))  # 12^n
    qps = rng.uniform(5, 60, 6)
    win = tables.window_arrays(qps, rng.integers(256, 4096, 6), 0, rng.uniform(0.02, 0.6, 6))
    gpu = _native.plan_windows_host(abi.MODE_ORACLE, prob, win, grid=grid)
    cpu = orc.plan_windows(abi.MODE_ORACLE, prob, win, grid=grid)
    for f in tables.DecisionArrays.FIELDS:
        assert getattr(gpu, f).tobytes() == getattr(cpu, f).tobytes(), (shape, n, f)
    assert gpu.feasible.any()


def test_multimodal_12op_exhaustive_vs_oracle(nat_loaded, orc):
    """cfg3: 12 operators, (P in {1,2}, R<=3, B=1)^12 = 2.2e9 candidates per window."""
    from paper_2511_02248_b200 import _native
    prob = tables.pack_problem(*scenarios.scenario("cfg3"))
    g = scenarios.GRIDS["cfg3"]
    grid = tables.pack_grid(prob, model.AutoscaleParams(slo=1.0), model.BruteForceBounds(**g))
    tw = scenarios.trace_windows("cfg3")
    idx = np.array([3, 30])
    for phase in ("prefill", "decode"):
        win = tables.window_arrays(tw[phase + "_qps"][idx], tw[phase + "_len"][idx],
                                   tables.PHASE_INDEX[phase], scenarios.SLO["cfg3"][phase])
        gpu = _native.plan_windows_host(abi.MODE_ORACLE, prob, win, grid=grid)
        cpu = orc.plan_windows(abi.MODE_ORACLE, prob, win, grid=grid)
        for f in tables.DecisionArrays.FIELDS:
            assert getattr(gpu, f).tobytes() == getattr(cpu, f).tobytes(), (phase, f)


@pytest.fixture(scope="module")
def nat_loaded():
    from paper_2511_02248_b200 import _native
    _native.load()
    assert _native.device_count() >= 1
    return _native


@pytest.mark.parametrize("p_of", [
    {"down": (1,), "lm_head": (1, 2)},             # k menu 3 < j tile 6 (padded register k tile)
    {"down": (1, 2), "lm_head": (1,)},             # j menu 3 -> tile 4, k menu 6 > 4 (shared k loop)
    {"act": (1,), "down": (1, 2, 4), "lm_head": (2, 4)},  # k 9 / j 6
])
def test_ragged_menus_70b_vs_oracle(nat_loaded, orc, p_of):
    """Per-operator parallelism dicts give the k / j levels different menu
    sizes: the register k tile with +inf padding, and the shared-memory k loop
    next to a small j tile, against the oracle on the 10-op 70B chain."""
    from paper_2511_02248_b200 import _native
    dag, prof = scenarios.scenario("cfg2")
    prob = tables.pack_problem(dag, prof)
    par = {op: p_of.get(op, (1, 2)) for op in prob.ids}
    params = model.AutoscaleParams(slo=1.0, parallelism=par, b_max=1)
    grid = tables.pack_grid(prob, params, model.BruteForceBounds(r_max=3))
    tw = scenarios.trace_windows("cfg2")
    idx = np.array([0, 7, 19, 33, 58])
    n_feasible = 0
    for phase in ("prefill", "decode"):
        for scale in (1.0, 4.0):  # the scenario SLO and a loose one (feasible decisions to compare)
            win = tables.window_arrays(tw[phase + "_qps"][idx], tw[phase + "_len"][idx],
                                       tables.PHASE_INDEX[phase], scale * scenarios.SLO["cfg2"][phase])
            gpu = _native.plan_windows_host(abi.MODE_ORACLE, prob, win, grid=grid)
            cpu = orc.plan_windows(abi.MODE_ORACLE, prob, win, grid=grid)
            for f in tables.DecisionArrays.FIELDS:
                assert getattr(gpu, f).tobytes() == getattr(cpu, f).tobytes(), (phase, scale, f)
            n_feasible += int(cpu.feasible.sum())
    assert n_feasible > 0
