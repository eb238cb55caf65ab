"""The fused per-window entry points give the same bytes as the separate ones.

opsc_menu_stability = opsc_menu_build + opsc_stability_check and
opsc_decode_materialize = opsc_menu_fallback + opsc_decode_decisions +
opsc_materialize(config_order 0) (include/opscale_b200.h). The planners use
the fused forms; the separate entry points stay in the ABI, so both chains
run here on the same windows -- feasible winners, SLOs no candidate meets
(the per-op fallback), idle windows, and arrival rates past every replica
bound (NoStableConfig from the bounds and from the pre-check) -- and every
decision array must match.
"""

import numpy as np
import pytest

from paper_2511_02248_b200 import abi, model, tables

pytestmark = pytest.mark.gpu


def _windows(name):
    from workloads import scenarios
    dag, prof = scenarios.scenario(name)
    tw = scenarios.trace_windows(name)
    slo = scenarios.SLO[name]["prefill"]
    idx = np.arange(12) % len(tw["prefill_qps"])  # cfg1 has one window: repeat it
    q = np.asarray(tw["prefill_qps"], dtype=np.float64)[idx].copy()
    L = np.asarray(tw["prefill_len"])[idx].copy()
    q[3] = 0.0          # idle
    q[5] = 1e9          # past every replica bound
    win = tables.window_arrays(q, L, 0, slo)
    win = win.take(np.arange(win.n))
    win.slo[7] = slo * 1e-6  # no candidate meets it: per-op fallback
    win.slo[8] = np.inf
    return dag, prof, win, model.BruteForceBounds(**scenarios.GRIDS[name]), model.AutoscaleParams(slo=slo)


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3"])
def test_fused_chain_matches_separate(name):
    import torch

    from paper_2511_02248_b200 import _native as nat
    from paper_2511_02248_b200 import device
    dag, prof, win, bounds, params = _windows(name)
    prob = tables.pack_problem(dag, prof)
    grid = tables.pack_grid(prob, params, bounds)
    L = nat.load()
    r = nat.ref

    fused = device.DevicePlanner(prob, win, abi.MODE_ORACLE, grid=grid)
    fused.step()
    want = fused.decisions()

    sep = device.DevicePlanner(prob, win, abi.MODE_ORACLE, grid=grid)
    s = torch.cuda.current_stream().cuda_stream
    st = sep.out_t["status"].data_ptr()
    sep._init()
    nat.check(L.opsc_menu_build(r(prob.table), r(grid), sep.win, sep.menu.data_ptr(), st, s), "menu")
    nat.check(L.opsc_stability_check(r(prob.table), r(grid), sep.win, st, s), "stability")
    sep.compose()
    nat.check(L.opsc_menu_fallback(r(prob.table), r(grid), sep.W, sep.menu.data_ptr(), sep.fb.data_ptr(), s), "fb")
    nat.check(L.opsc_decode_decisions(r(prob.table), r(grid), sep.W, sep.key.data_ptr(), sep.fb.data_ptr(),
                                      sep.out_t["cfg"].data_ptr(), sep.out_t["feasible"].data_ptr(), st, s), "dec")
    nat.check(L.opsc_materialize(r(prob.table), sep.win, 0, r(sep.dplace), sep.out, s), "mat")
    got = sep.decisions()
    for f in tables.DecisionArrays.FIELDS:
        assert getattr(got, f).tobytes() == getattr(want, f).tobytes(), f
    # the crafted windows really took the paths they were made for
    assert want.status[3] & abi.W_IDLE
    assert not want.feasible[7] and not (want.status[7] & abi.W_NO_STABLE_BOUNDS)
    assert want.status[5] & (abi.W_NO_STABLE_BOUNDS | abi.W_NO_STABLE_PARAMS)
    assert want.feasible.sum() >= 1
