"""Device-resident planning pipeline (torch owns the HBM buffers).

`DevicePlanner` keeps a batch of windows resident in HBM and runs the search
kernels through the device-pointer C-ABI entry points on torch's current
stream. It is what bench.py times (`value`) and what the multi-GPU path
shards: every rank enumerates its slice of each window's candidate space and
one MIN all-reduce of the packed (objective << 40 | lexicographic index) keys
yields the global decision -- the same merge the single-GPU kernel does with
atomicMin, so the decision is identical for any number of ranks.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _native, abi, tables


class DevicePlanner:
    def __init__(self, problem, windows: tables.WindowArrays, mode=abi.MODE_ORACLE, grid=None,
                 model=None, place=None, device="cuda", greedy=None, trace_cap=1024):
        self.problem, self.mode = problem, mode
        self.grid = grid if grid is not None else abi.OpscGrid()
        self.model = model if model is not None else abi.OpscModelSpec()
        self.greedy = greedy if greedy is not None else abi.OpscGreedySpec()
        self.place = place or tables.pack_place()
        self.dev = torch.device(device)
        self.L = _native.load()
        n = problem.n_ops
        if isinstance(windows, dict):
            # window SoA already resident in HBM (e.g. straight from windowize_device)
            self.win_t = {k: windows[k].to(self.dev).contiguous()
                          for k in ("qps", "seq_len", "phase", "slo", "eps")}
            W = int(self.win_t["qps"].numel())
        else:
            W = windows.n
            to = lambda a: torch.from_numpy(np.array(a, copy=True)).to(self.dev)
            self.win_t = {k: to(getattr(windows, k)) for k in ("qps", "seq_len", "phase", "slo", "eps")}
        self.W, self.n = W, n
        self.win = abi.OpscWindows()
        self.win.n = W
        for k, t in self.win_t.items():
            setattr(self.win, k, t.data_ptr())
        E = self.grid.menu_off[n] if mode == abi.MODE_ORACLE else 0
        self.E = E
        z = lambda *shape, dt: torch.zeros(shape, dtype=dt, device=self.dev)
        self.menu = z(max(W * E, 1), dt=torch.float64)
        self.fb = z(max(W * n, 1), dt=torch.int32)
        self.key = z(W, dt=torch.int64)
        self.out_t = {
            "key": self.key, "cfg": z(W, n, 3, dt=torch.int16), "feasible": z(W, dt=torch.uint8),
            "status": z(W, dt=torch.int32), "latency": z(W, dt=torch.float64),
            "objective": z(W, dt=torch.int32), "path": z(W, n, dt=torch.int8),
            "pred": z(W, n, abi.PRED_FIELDS, dt=torch.float64), "stable": z(W, n, dt=torch.uint8),
            "energy": z(W, dt=torch.float64), "memory": z(W, dt=torch.float64),
            "devices": z(W, dt=torch.int32),
        }
        self.out = abi.OpscDecisions()
        for k, t in self.out_t.items():
            setattr(self.out, k, t.data_ptr())
        # operator mode: uniform reseed inputs + move trace
        self.trace_cap = trace_cap if mode == abi.MODE_OPERATOR else 0
        self.u_cfg = z(W, n, 3, dt=torch.int16)
        self.u_feas = z(W, dt=torch.uint8)
        self.u_status = z(W, dt=torch.int32)
        self.trace_len = z(W, dt=torch.int32)
        self.trace = z(max(W * self.trace_cap * tables.TRACE_DTYPE.itemsize, 1), dt=torch.uint8)
        self.out.trace_cap = self.trace_cap
        self.out.trace_len = self.trace_len.data_ptr()
        self.out.trace = self.trace.data_ptr()
        caps = torch.from_numpy(self.place.mem_cap).to(self.dev)
        self._caps = caps
        self.dplace = abi.OpscPlaceSpec()
        for f, _ in abi.OpscPlaceSpec._fields_:
            setattr(self.dplace, f, getattr(self.place.spec, f))
        self.dplace.mem_cap = caps.data_ptr()
        self.launches = 0

    def _s(self):
        return torch.cuda.current_stream(self.dev).cuda_stream

    def _ck(self, rc, what):
        _native.check(rc, what)
        self.launches += 1

    def _init(self, reset_key=True):
        # status = idle bit for qps <= 0, keys = +inf, feasible = 0
        self._ck(self.L.opsc_init_windows(self.win, self.out_t["status"].data_ptr(),
                                          self.key.data_ptr() if reset_key else None,
                                          self.out_t["feasible"].data_ptr(), self._s()), "init_windows")

    def menus(self):
        """K1 menus + K1b stability pre-check, one fused launch."""
        r = _native.ref
        self._ck(self.L.opsc_menu_stability(r(self.problem.table), r(self.grid), self.win,
                                            self.menu.data_ptr(), self.out_t["status"].data_ptr(),
                                            self._s()), "menu_stability")

    def compose(self, shard=0, n_shards=1):
        r = _native.ref
        self._ck(self.L.opsc_compose_argmin(r(self.problem.table), r(self.grid), self.win,
                                            self.menu.data_ptr(), shard, n_shards,
                                            self.key.data_ptr(), self._s()), "compose_argmin")

    def certify(self, band_ulps=abi.CERTIFY_BAND_ULPS):
        """Opt-in summation-order certificate (brute force, after compose):
        ORs W_ORDER_SENSITIVE into status where argmin over lat <= slo - band
        and argmin over lat <= slo + band differ (opsc_certify_order)."""
        if self.mode != abi.MODE_ORACLE:
            return
        if getattr(self, "_cert_ws", None) is None:
            nb = int(self.L.opsc_certify_workspace(self.W))
            self._cert_ws = torch.empty(max(nb, 1), dtype=torch.uint8, device=self.dev)
        r = _native.ref
        self._ck(self.L.opsc_certify_order(r(self.problem.table), r(self.grid), self.win,
                                           self.menu.data_ptr(), float(band_ulps),
                                           self._cert_ws.data_ptr(), self._cert_ws.numel(),
                                           self.out_t["status"].data_ptr(), self._s()), "certify_order")

    def finish(self):
        r, s = _native.ref, self._s()
        if self.mode == abi.MODE_ORACLE:
            # fallback + decode fused into the materialisation launch
            self._ck(self.L.opsc_decode_materialize(r(self.problem.table), r(self.grid), self.win,
                                                    self.key.data_ptr(), self.menu.data_ptr(),
                                                    r(self.dplace), self.out, s), "decode_materialize")
            return
        order = 1
        self._ck(self.L.opsc_materialize(r(self.problem.table), self.win, order, r(self.dplace),
                                         self.out, s), "materialize")

    def operator(self):
        """greedy_autoscale. The model-level reseed candidates (K3) are
        computed on a side stream concurrently with greedy phase 1 (init +
        first loop); phase 2 (reseed, headroom, prune) joins both."""
        r = _native.ref
        if not hasattr(self, "_side"):
            self._side = torch.cuda.Stream(self.dev)
            nb = self.L.opsc_greedy_state_bytes(self.W)
            self._gstate = torch.empty(max(nb, 1), dtype=torch.uint8, device=self.dev)
        main = torch.cuda.current_stream(self.dev)
        self._side.wait_stream(main)
        side = self._side.cuda_stream
        self._ck(self.L.opsc_init_windows(self.win, self.u_status.data_ptr(), None,
                                          self.u_feas.data_ptr(), side), "init_windows")
        # the reseed runs beside phase 1; tabulated (B, R) points: a 70B prefill
        # window's K3 took 129 us in the one-kernel form, more than phase 1
        self._model_grid_into(self.greedy.model, self.u_cfg, self.u_feas, self.u_status, side)
        args = (r(self.problem.table), r(self.greedy), self.win)
        uni = (self.u_cfg.data_ptr(), self.u_feas.data_ptr(), self.u_status.data_ptr())
        self._ck(self.L.opsc_greedy_phase(*args, 1, self._gstate.data_ptr(), *uni, self.out,
                                          main.cuda_stream), "greedy_phase1")
        main.wait_stream(self._side)
        self._ck(self.L.opsc_greedy_phase(*args, 2, self._gstate.data_ptr(), *uni, self.out,
                                          main.cuda_stream), "greedy_phase2")

    # small batches tabulate every (B, R) point in parallel (csrc/k_model.cu)
    MODEL_TABLE_POINTS = 1 << 22

    def _model_grid_into(self, spec, cfg, feas, status, stream, table=True):
        r = _native.ref
        pts = self.W * spec.b_cap * spec.r_cap * self.n
        if table and pts <= self.MODEL_TABLE_POINTS:
            nb = self.L.opsc_model_table_bytes(r(spec), self.W, self.n)
            if getattr(self, "_mtab", None) is None or self._mtab.numel() < nb:
                self._mtab = torch.empty(nb, dtype=torch.uint8, device=self.dev)
            self._ck(self.L.opsc_model_grid_table(r(self.problem.table), r(spec), self.win,
                                                  cfg.data_ptr(), feas.data_ptr(), status.data_ptr(),
                                                  self._mtab.data_ptr(), self._mtab.numel(), stream),
                     "model_grid_table")
        else:
            self._ck(self.L.opsc_model_grid(r(self.problem.table), r(spec), self.win, cfg.data_ptr(),
                                            feas.data_ptr(), status.data_ptr(), stream), "model_grid")

    def model_grid(self):
        self._model_grid_into(self.model, self.out_t["cfg"], self.out_t["feasible"],
                              self.out_t["status"], self._s())

    def step(self, shard=0, n_shards=1, allreduce=None, compose_events=None, merge=None, certify=False):
        """One pass of the hot path over the resident batch of windows.
        `merge` (dist.PeerMerge): the multi-GPU merge fused into the compose
        kernel over peer memory instead of `allreduce` after it. `certify`:
        also run the summation-order certificate (single GPU)."""
        if merge is not None and self.mode == abi.MODE_ORACLE:
            return merge.step(self, compose_events)
        self._init()
        if self.mode == abi.MODE_ORACLE:
            self.menus()
            if compose_events:
                compose_events[0].record()
            self.compose(shard, n_shards)
            if compose_events:
                compose_events[1].record()
            if allreduce is not None:
                allreduce(self.key)
            if certify:
                self.certify()
        elif self.mode == abi.MODE_OPERATOR:
            self.operator()
        else:
            self.model_grid()
        self.finish()

    def capture(self, shard=0, n_shards=1, allreduce=None):
        """Record one step into a CUDA graph (after a warm-up step that creates
        the lazily allocated workspaces). Update `win_t` in place, then
        `graph.replay()` re-plans the resident windows with one launch."""
        self.step(shard, n_shards, allreduce)
        torch.cuda.synchronize(self.dev)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self.step(shard, n_shards, allreduce)
        return g

    def load_windows(self, host: tables.WindowArrays):
        """Async H2D of a host window SoA (pinned for overlap) into the
        resident buffers, on the current stream."""
        for k, t in self.win_t.items():
            a = getattr(host, k)
            t.copy_(torch.from_numpy(a.view(np.int32) if a.dtype == np.uint32 else a), non_blocking=True)

    def fetch(self, host: tables.DecisionArrays, sync=True):
        """D2H of the decisions into a (pinned) host DecisionArrays on the
        current stream; waits for it unless `sync` is False (the caller then
        synchronises before reading `host`)."""
        for k, t in self.out_t.items():
            a = getattr(host, k)
            dst = torch.from_numpy(a.view(np.int32) if a.dtype == np.uint32 else a)
            dst.copy_(t.view(dst.shape), non_blocking=True)
        if sync:
            torch.cuda.current_stream(self.dev).synchronize()
        return host

    def decisions(self) -> tables.DecisionArrays:
        torch.cuda.synchronize(self.dev)
        out = tables.DecisionArrays(self.W, self.n, self.trace_cap)
        for k, t in self.out_t.items():
            getattr(out, k)[...] = t.cpu().numpy().astype(getattr(out, k).dtype).reshape(
                getattr(out, k).shape)
        if self.trace_cap:
            out.trace_len[...] = self.trace_len.cpu().numpy()
            out.trace[...] = self.trace.cpu().numpy().view(tables.TRACE_DTYPE).reshape(
                self.W, self.trace_cap)
        return out


def fp64_peak(iters=20000):
    """Measured FP64 (DADD) issue peak of this GPU, op/s (live microbenchmark)."""
    L = _native.load()
    ms, ops = C.c_float(), C.c_double()
    _native.check(L.opsc_fp64_peak(iters, C.cast(C.byref(ms), C.c_void_p),
                                   C.cast(C.byref(ops), C.c_void_p),
                                   torch.cuda.current_stream().cuda_stream), "fp64_peak")
    return ops.value / (ms.value * 1e-3)
