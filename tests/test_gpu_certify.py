"""Opt-in summation-order certificate (OPSC_W_ORDER_SENSITIVE).

The reference's brute-force leaf test sums path weights over a frozenset
(autoscaler.py:765, 792-796), so its order -- and, for candidates within a
few ulps of the SLO, its verdict -- depends on PYTHONHASHSEED. The
certificate flags a window when argmin over {lat <= slo - band} differs from
argmin over {lat <= slo + band}. Checked here:

* opsc_certify_order on crafted tie menus against the CPU oracle's literal
  enumeration at the two shifted SLOs (several bands, chain and fork DAGs);
* the planner API (decide_windows(certify=True), host-buffer C-ABI call):
  decisions bit-identical to the uncertified call, only the status bit
  added; unflagged on the bench workloads (as tools/boundary_check.py found
  no candidate within 64 ulps there); flagged when the SLO is set to the
  winner's own latency or one ulp below it.
"""

import numpy as np
import pytest

from paper_2511_02248_b200 import abi, model, tables

from test_gpu_compose_edges import _dag, _menus

pytestmark = pytest.mark.gpu


def _shifted(win, band_ulps):
    lo, hi = win.take(np.arange(win.n)), win.take(np.arange(win.n))
    for w in range(win.n):
        s = float(win.slo[w])
        band = band_ulps * (np.nextafter(s, np.inf) - s) if np.isfinite(s) else 0.0
        lo.slo[w], hi.slo[w] = s - band, s + band
    return lo, hi


@pytest.mark.parametrize("shape,n", [("chain", 5), ("fork", 6)])
def test_certify_order_vs_oracle(orc, shape, n):
    import torch

    from paper_2511_02248_b200 import _native as nat
    nat.load()
    rng = np.random.default_rng(11 + n)
    prob = _dag(n, shape)
    grid = tables.pack_grid(prob, model.AutoscaleParams(slo=1.0),
                            model.BruteForceBounds(r_max=3, b_max=2, parallelism=(1, 2)))
    slos = [1.0, 0.7, 0.3 + 1e-13, 2.5, 0.9999999999999999, np.inf]
    W = len(slos)
    win = tables.window_arrays(np.full(W, 10.0), np.full(W, 512), 0, 1.0)
    win.slo[:] = slos
    mw = _menus(rng, prob, grid, slos, "tie" if shape == "chain" else "short")
    dev = torch.device("cuda:0")
    t = {k: torch.from_numpy(np.ascontiguousarray(getattr(win, k))).to(dev)
         for k in ("qps", "seq_len", "phase", "slo", "eps")}
    dw = abi.OpscWindows()
    dw.n = W
    for k in t:
        setattr(dw, k, t[k].data_ptr())
    mwd = torch.from_numpy(mw).to(dev)
    L = nat.load()
    ws = torch.empty(int(L.opsc_certify_workspace(W)), dtype=torch.uint8, device=dev)
    flagged_any = False
    # the tie menus sit on a 2^-40 grid: 4096 ulps of slo = 1.0 is one grain
    for band in (0.0, 64.0, 4096.0, 3 * 4096.0, 1e6):
        status = torch.zeros(W, dtype=torch.int32, device=dev)
        nat.check(L.opsc_certify_order(nat.ref(prob.table), nat.ref(grid), dw, mwd.data_ptr(), band,
                                       ws.data_ptr(), ws.numel(), status.data_ptr(),
                                       torch.cuda.current_stream().cuda_stream), "certify")
        got = (status.cpu().numpy() & abi.W_ORDER_SENSITIVE) != 0
        lo, hi = _shifted(win, band)
        want = orc.compose(prob, grid, lo, mw) != orc.compose(prob, grid, hi, mw)
        assert (got == want).all(), (band, got, want)
        flagged_any |= bool(got.any())
        if band == 0.0:
            assert not got.any()
    assert flagged_any


def _cfg(name):
    from workloads import scenarios
    dag, prof = scenarios.scenario(name)
    tw = scenarios.trace_windows(name)
    bounds = model.BruteForceBounds(**scenarios.GRIDS[name])
    params = model.AutoscaleParams(slo=scenarios.SLO[name]["prefill"])
    return dag, prof, tw, bounds, params


@pytest.mark.parametrize("name,step", [("cfg1", 1), ("cfg5", 97)])
def test_certified_decisions_unchanged_and_clear(name, step):
    from paper_2511_02248_b200 import planners
    dag, prof, tw, bounds, params = _cfg(name)
    idx = range(0, len(tw["prefill_qps"]), step)
    pts = [model.WorkloadPoint(float(tw["prefill_qps"][i]), int(tw["prefill_len"][i]), "prefill")
           for i in idx if tw["prefill_qps"][i] > 0]
    plain = planners.decide_windows(dag, prof, pts, params, "oracle", bounds)
    cert = planners.decide_windows(dag, prof, pts, params, "oracle", bounds, certify=True)
    for a, b in zip(plain, cert):
        for f in tables.DecisionArrays.FIELDS:
            x, y = getattr(a.arrays, f), getattr(b.arrays, f)
            if f == "status":
                assert ((y & ~np.uint32(abi.W_ORDER_SENSITIVE)) == x).all()
            else:
                assert x.tobytes() == y.tobytes(), f
        # bench workloads: no candidate near the SLO, nothing flagged
        assert not any(b.order_sensitive(k) for k in range(len(b)))


def test_slo_at_winner_latency_is_flagged():
    """SLO = the winner's own iteration latency (and one ulp below it): the
    winner sits on the mask boundary, so some summation order could reject
    it (or accept a cheaper neighbour) -- the certificate must say so."""
    from paper_2511_02248_b200 import planners
    dag, prof, tw, bounds, params = _cfg("cfg1")
    pt = model.WorkloadPoint(float(tw["prefill_qps"][0]), int(tw["prefill_len"][0]), "prefill")
    base = planners.brute_force_autoscale(dag, prof, pt, params, bounds, guards=False)
    assert base.feasible
    lat = base.iteration_latency
    at = model.AutoscaleParams(slo=lat)
    below = model.AutoscaleParams(slo=float(np.nextafter(lat, 0.0)))
    res = {}
    for tag, prm in (("at", at), ("below", below)):
        [dec] = planners.decide_windows(dag, prof, [pt], prm, "oracle", bounds, certify=True)
        res[tag] = dec.order_sensitive(0)
        [dec0] = planners.decide_windows(dag, prof, [pt], prm, "oracle", bounds)
        assert dec.plan(0) == dec0.plan(0)
    assert res["at"] and res["below"], res


def test_certify_host_buffer_matches_device_path():
    """The C-ABI host-buffer call with OPSC_PLAN_CERTIFY and the device-pointer
    pipeline (DevicePlanner.step(certify=True)) give identical bytes."""
    from paper_2511_02248_b200 import _native, device
    dag, prof, tw, bounds, params = _cfg("cfg1")
    prob = tables.pack_problem(dag, prof)
    grid = tables.pack_grid(prob, params, bounds)
    qps = np.asarray(tw["prefill_qps"][:8], dtype=np.float64)
    win = tables.window_arrays(qps, np.asarray(tw["prefill_len"][:8]), 0, params.slo)
    # put half the windows on a boundary: slo = some candidate's latency
    ref = _native.plan_windows_host(abi.MODE_ORACLE, prob, win, grid=grid)
    win = win.take(np.arange(win.n))  # own, writable copies
    win.slo[::2] = ref.latency[::2]
    host = _native.plan_windows_host(abi.MODE_ORACLE, prob, win, grid=grid, certify=True)
    dp = device.DevicePlanner(prob, win, abi.MODE_ORACLE, grid=grid)
    dp.step(certify=True)
    got = dp.decisions()
    for f in tables.DecisionArrays.FIELDS:
        assert getattr(host, f).tobytes() == getattr(got, f).tobytes(), f
    assert (host.status[::2] & abi.W_ORDER_SENSITIVE).all()
