"""GPU windowize (csrc/k_windowize.cu) against the reference-generated window
statistics (workloads/traces.npz) and the CPU oracle on unsorted / edge traces."""

import numpy as np
import pytest

from paper_2511_02248_b200 import workload
from workloads import scenarios

pytestmark = pytest.mark.gpu


def _records(cfg):
    spec = scenarios.TRACES[cfg]
    recs = workload.synth_workload(workload.SynthSpec(**spec["spec"]), spec["seed"])
    return (np.array([r.arrival_time for r in recs]), np.array([r.input_len for r in recs]),
            np.array([r.output_len for r in recs]), spec)


@pytest.mark.parametrize("cfg", ["cfg1", "cfg2", "cfg3", "cfg5"])
def test_windowize_matches_reference(cfg):
    arr, li, lo, spec = _records(cfg)
    pq, pl, dq = (x.cpu().numpy() for x in workload.windowize_device(
        arr, li, lo, spec["window_len"], spec["quantile"]))
    tw = scenarios.trace_windows(cfg)
    assert np.array_equal(pq, tw["prefill_qps"])
    assert np.array_equal(pl, tw["prefill_len"])
    assert np.array_equal(dq, tw["decode_qps"])


def test_windowize_unsorted_and_edges(orc):
    rng = np.random.default_rng(11)
    for trial in range(20):
        n = int(rng.integers(1, 5000))
        arr = rng.uniform(0, rng.uniform(1, 4000), n)
        if trial % 4 == 0:
            arr[: n // 2] = np.floor(arr[: n // 2] / 60.0) * 60.0  # exact window boundaries
        li = rng.integers(1, 1 << int(rng.integers(1, 22)), n)
        lo = rng.integers(0, 3000, n)
        wl = float(rng.choice([1.0, 7.5, 60.0, 300.0]))
        q = float(rng.choice([0.5, 0.95, 0.99, 1.0, 1e-9]))
        exp = orc.windowize(arr, li, lo, wl, q)
        got = [x.cpu().numpy() for x in workload.windowize_device(arr, li, lo, wl, q)]
        for a, b in zip(got, exp):
            assert np.array_equal(a, b), (trial, n, wl, q)


def test_windowize_points_api():
    recs = workload.synth_workload(workload.SynthSpec(kind="burst", rate=5.0, duration=900.0), 3)
    assert workload.windowize_points(recs, 60.0, 0.9) == workload.windowize(recs, 60.0, 0.9)
    assert workload.windowize_points([], 60.0) == []
