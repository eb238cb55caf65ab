"""Summation-order certificate (dev/evidence tool, GPU): per window, the
number of candidates whose canonical critical-path latency lies within
BAND ulps of the SLO. Only those could change feasibility under the
reference's frozenset-ordered, Neumaier-compensated leaf sum
(autoscaler.py:792-794); a zero count makes the window's decision
independent of PYTHONHASHSEED. Writes gpurun_out/r01_boundary.json (kept as profiles/r01_boundary.json).

    python tools/boundary_check.py [band_ulps]
"""
import json
import os
import sys
import time

import numpy as np
import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
from paper_2511_02248_b200 import _native, abi, model, tables  # noqa: E402
from workloads import scenarios  # noqa: E402

BAND = float(sys.argv[1]) if len(sys.argv) > 1 else 64.0
L = _native.load()
dev = torch.device("cuda:0")
s = torch.cuda.current_stream().cuda_stream
out = {"band_ulps": BAND, "workloads": {}}
for cfg, phases in (("cfg5", ("prefill",)), ("cfg2", ("prefill", "decode")), ("cfg1", ("prefill", "decode"))):
    prob = tables.pack_problem(*scenarios.scenario(cfg))
    grid = tables.pack_grid(prob, model.AutoscaleParams(slo=1.0), model.BruteForceBounds(**scenarios.GRIDS[cfg]))
    tw = scenarios.trace_windows(cfg)
    for ph in phases:
        win = tables.window_arrays(tw[ph + "_qps"], tw[ph + "_len"], tables.PHASE_INDEX[ph], scenarios.SLO[cfg][ph])
        t = {k: torch.from_numpy(np.ascontiguousarray(getattr(win, k))).to(dev)
             for k in ("qps", "seq_len", "phase", "slo", "eps")}
        dw = abi.OpscWindows()
        dw.n = win.n
        for k in t:
            setattr(dw, k, t[k].data_ptr())
        E = grid.menu_off[prob.n_ops]
        mw = torch.empty((win.n, E), dtype=torch.float64, device=dev)
        st = torch.zeros(win.n, dtype=torch.int32, device=dev)
        _native.check(L.opsc_menu_build(_native.ref(prob.table), _native.ref(grid), dw, mw.data_ptr(),
                                        st.data_ptr(), s), "menu")
        cnt = torch.zeros(win.n, dtype=torch.int64, device=dev)
        t0 = time.perf_counter()
        _native.check(L.opsc_compose_boundary(_native.ref(prob.table), _native.ref(grid), dw, mw.data_ptr(),
                                              BAND, cnt.data_ptr(), s), "boundary")
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        c = cnt.cpu().numpy()
        space = int(np.prod([grid.menu_off[v + 1] - grid.menu_off[v] for v in range(prob.n_ops)]))
        rec = {"windows": int(win.n), "candidates": space * int(win.n),
               "windows_with_boundary_candidates": int((c > 0).sum()), "boundary_candidates": int(c.sum()),
               "seconds": dt}
        out["workloads"][f"{cfg}/{ph}"] = rec
        print(cfg, ph, rec, flush=True)
os.makedirs(os.path.join(REPO, "gpurun_out"), exist_ok=True)  # copied to profiles/ by hand
json.dump(out, open(os.path.join(REPO, "gpurun_out", "r01_boundary.json"), "w"), indent=1)
