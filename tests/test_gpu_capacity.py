"""Config 4 (throughput under a fixed 8-GPU budget): the GPU search equals
the same search driven by the CPU oracle, bit for bit (parity against the
reference is unpinned: the reference has no such operation)."""

import numpy as np
import pytest

from paper_2511_02248_b200 import abi, capacity, model, tables
from workloads import scenarios

pytestmark = pytest.mark.gpu


def _oracle_eval(orc, m, prob, grid, spec, greedy, place):
    def evaluate(win):
        return orc.plan_windows(m, prob, win, grid=grid, model=spec, place=place, greedy=greedy, trace_cap=0)
    return evaluate


@pytest.mark.parametrize("mode,cfg,k", [("oracle", "cfg1", 5), ("model", "cfg2", 6), ("operator", "cfg2", 3)])
def test_capacity_gpu_equals_oracle(orc, mode, cfg, k):
    dag, prof = scenarios.scenario(cfg)
    tw = scenarios.trace_windows("cfg2")
    idx = np.linspace(0, 59, k).round().astype(int)
    pts = [model.WorkloadPoint(float(tw["prefill_qps"][i]), int(tw["prefill_len"][i]), "prefill") for i in idx]
    params = model.AutoscaleParams(slo=scenarios.SLO[cfg]["prefill"])
    bounds = model.BruteForceBounds(**scenarios.GRIDS[cfg]) if mode == "oracle" else None
    kw = dict(mode=mode, bounds=bounds, budget=8, mem_cap=80e9, fan=16, rel_tol=1e-5, max_rounds=8)
    gpu = capacity.max_qps_under_budget(dag, prof, pts, params, **kw)
    prob = tables.pack_problem(dag, prof)
    m = capacity._MODES[mode]
    ev = _oracle_eval(orc, m, prob, tables.pack_grid(prob, params, bounds) if mode == "oracle" else None,
                      tables.pack_model(prob, params),
                      tables.pack_greedy(prob, params) if mode == "operator" else None,
                      tables.pack_place(model.make_fleet(8, 80e9)))
    cpu = capacity.max_qps_under_budget(dag, prof, pts, params, evaluate=ev, **kw)
    for f in ("qps", "upper", "cfg", "devices", "objective", "latency"):
        assert getattr(gpu, f).tobytes() == getattr(cpu, f).tobytes(), f
    assert (gpu.qps > 0).all() and (gpu.devices <= 8).all()
