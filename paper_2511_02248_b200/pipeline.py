"""Trace -> decisions, resident in HBM end to end.

The reference's per-trace flow (cli.cmd_autoscale, cli.py:123-186) is:
windowize the trace (workload.py:114-158), then plan every window and phase
(runner.run_point -> plan_for_mode). Here the records go to the device once;
windowing (K7), planning (K1-K5) and materialisation (K4) then run without
leaving HBM, and only the decisions come back.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _native, abi, device, model, tables, workload
from .plans import WindowDecisions

_MODES = {"oracle": abi.MODE_ORACLE, "model": abi.MODE_MODEL, "operator": abi.MODE_OPERATOR}


class TracePlanner:
    """Plans every window of a trace for both phases (prefill: TTFT SLO,
    decode: TBT SLO, as cli.py:114-120 maps them)."""

    def __init__(self, dag, profiles, params_by_phase, mode="operator", bounds=None,
                 window_len=60.0, quantile=0.95, device_="cuda", trace_cap=1024):
        self.problem = tables.pack_problem(dag, profiles)
        self.params = params_by_phase
        self.mode = _MODES[mode] if isinstance(mode, str) else mode
        self.bounds = bounds if bounds is not None else model.BruteForceBounds()
        self.window_len, self.quantile = window_len, quantile
        self.dev = torch.device(device_)
        self.trace_cap = trace_cap
        self.planners = {}
        for ph in ("prefill", "decode"):
            self.problem.require_phase(ph)

    def _specs(self, ph):
        p = self.params[ph]
        grid = tables.pack_grid(self.problem, p, self.bounds) if self.mode == abi.MODE_ORACLE else None
        spec = tables.pack_model(self.problem, p)
        greedy = tables.pack_greedy(self.problem, p) if self.mode == abi.MODE_OPERATOR else None
        return grid, spec, greedy

    def run(self, arrival, input_len, output_len):
        """Device pipeline over one trace; returns {phase: DevicePlanner} with
        decisions resident on the device (call .decisions() to fetch)."""
        pq, pl, dq = workload.windowize_device(arrival, input_len, output_len, self.window_len,
                                               self.quantile, self.dev)
        W = int(pq.numel())
        out = {}
        for ph, qps, ln in (("prefill", pq, pl), ("decode", dq, torch.ones_like(pl))):
            p = self.params[ph]
            win = {"qps": qps, "seq_len": ln,
                   "phase": torch.full((W,), tables.PHASE_INDEX[ph], dtype=torch.uint8, device=self.dev),
                   "slo": torch.full((W,), float(p.slo), dtype=torch.float64, device=self.dev),
                   "eps": torch.full((W,), float(p.epsilon), dtype=torch.float64, device=self.dev)}
            key = (ph, W)
            if key not in self.planners:
                grid, spec, greedy = self._specs(ph)
                self.planners[key] = device.DevicePlanner(self.problem, win, self.mode, grid=grid,
                                                          model=spec, greedy=greedy, device=self.dev,
                                                          trace_cap=self.trace_cap)
            pr = self.planners[key]
            for k in ("qps", "seq_len"):
                pr.win_t[k].copy_(win[k])
            pr.step()
            out[ph] = pr
        return out

    def plans(self, arrival, input_len, output_len):
        """[(prefill plan | None, decode plan | None)] per window (None for
        idle windows, which the CLI records as vacuous rows)."""
        res = self.run(arrival, input_len, output_len)
        decs = {}
        for ph, pr in res.items():
            arrays = pr.decisions()
            cut = np.nonzero(arrays.status & abi.W_TRACE_TRUNCATED)[0]
            if len(cut):  # move traces past trace_cap: re-plan those windows with room
                host = tables.WindowArrays(*(pr.win_t[k].cpu().numpy()[cut] for k in
                                             ("qps", "seq_len", "phase", "slo", "eps")))
                grid, spec, greedy = self._specs(ph)
                again = _native.plan_windows_host(self.mode, self.problem, host, grid=grid, model=spec,
                                                  greedy=greedy, trace_cap=int(arrays.trace_len[cut].max()))
                arrays = arrays.with_trace_cap(again.trace_cap)
                arrays.splice(cut, again)
            pts = [model.WorkloadPoint(max(float(q), 0.0), int(l), ph)
                   for q, l in zip(arrays_qps(pr), pr.win_t["seq_len"].cpu().numpy())]
            decs[ph] = WindowDecisions(self.problem, pts, arrays, self.mode,
                                       r_cap=self.params[ph].r_cap)
        W = len(decs["prefill"])
        return [(decs["prefill"].plan(i), decs["decode"].plan(i)) for i in range(W)]


def arrays_qps(planner):
    return planner.win_t["qps"].cpu().numpy()
