"""Config 4's capacity search logic (paper_2511_02248_b200/capacity.py) on a
synthetic evaluator: no device needed."""

import numpy as np

from paper_2511_02248_b200 import capacity, model, tables


def _threshold_eval(thr, n_ops=2):
    thr = np.asarray(thr, dtype=np.float64)

    def evaluate(win):
        # seq_len carries the window id in this synthetic test
        out = tables.DecisionArrays(win.n, n_ops)
        out.feasible[:] = (win.qps <= thr[win.seq_len - 1]).astype(np.uint8)
        out.devices[:] = 1
        out.objective[:] = np.round(win.qps).astype(np.int32)
        return out
    return evaluate


def test_search_brackets_a_monotone_threshold():
    thr = [37.25, 1e-9, 5e6, 0.3, 12.0]
    pts = [model.WorkloadPoint(10.0, i + 1, "prefill") for i in range(len(thr))]
    res = capacity.search(pts, model.AutoscaleParams(slo=1.0), _threshold_eval(thr), 2, budget=8,
                          fan=16, rel_tol=1e-6)
    for w, t in enumerate(thr):
        if t < 10.0 * 2.0 ** -8:  # below the smallest probed rate: capacity 0
            assert res.qps[w] == 0.0
            continue
        assert res.qps[w] <= t < res.upper[w]
        assert res.upper[w] - res.qps[w] <= 1e-6 * res.qps[w]
        assert res.objective[w] == round(res.qps[w])
    assert res.evaluated < 16 * len(thr) * res.rounds + 1


def test_search_respects_the_device_budget():
    def evaluate(win):
        out = tables.DecisionArrays(win.n, 1)
        out.feasible[:] = 1
        out.devices[:] = np.ceil(win.qps / 10.0).astype(np.int32)  # one device per 10 qps
        return out
    res = capacity.search([model.WorkloadPoint(3.0, 1, "decode")], model.AutoscaleParams(slo=1.0),
                          evaluate, 1, budget=8, fan=32, rel_tol=1e-9)
    assert res.qps[0] <= 80.0 < res.upper[0] and res.qps[0] > 80.0 * (1 - 1e-8)
    assert res.devices[0] == 8
