"""Synthetic traces and windowed demand (host side).

Same generators and windowing as the reference (workload.py:107-232):
Poisson thinning against the peak rate with numpy's default_rng, lognormal
input/output lengths, and per-window (prefill, decode) demand points with the
"higher" empirical quantile of input lengths. tests/test_host.py checks the
output bit-for-bit against the reference-generated fixture in workloads/traces.npz.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .model import WorkloadPoint


@dataclass(frozen=True)
class RequestRecord:
    arrival_time: float
    input_len: int
    output_len: int


@dataclass(frozen=True)
class SynthSpec:
    kind: str = "constant"  # constant | diurnal | burst
    rate: float = 10.0
    duration: float = 600.0
    input_len_median: float = 1024.0
    input_len_sigma: float = 0.5
    output_len_median: float = 256.0
    output_len_sigma: float = 0.3
    amplitude: float = 0.5
    period: float = 600.0
    burst_factor: float = 3.0
    burst_duty: float = 0.2

    def __post_init__(self):
        if self.kind not in ("constant", "diurnal", "burst"):
            raise ValueError(f"unknown workload kind {self.kind!r}")
        if self.rate <= 0 or self.duration <= 0:
            raise ValueError("rate and duration must be positive")
        if self.kind == "diurnal" and not (0.0 <= self.amplitude < 1.0):
            raise ValueError("diurnal amplitude must be in [0, 1)")
        if self.kind == "burst" and self.burst_factor < 1.0:
            raise ValueError("burst_factor must be >= 1")

    def rate_at(self, t: float) -> float:
        if self.kind == "diurnal":
            return self.rate * (1.0 + self.amplitude * math.sin(2.0 * math.pi * t / self.period))
        if self.kind == "burst":
            in_burst = (t % self.period) < self.burst_duty * self.period
            return self.rate * self.burst_factor if in_burst else self.rate
        return self.rate

    @property
    def peak_rate(self) -> float:
        if self.kind == "diurnal":
            return self.rate * (1.0 + self.amplitude)
        if self.kind == "burst":
            return self.rate * self.burst_factor
        return self.rate


def synth_workload(spec: SynthSpec, seed: int) -> list:
    """Deterministic synthetic trace: thinned Poisson arrivals at the peak
    rate, then lognormal lengths; draw order per accepted request is
    exponential, uniform, lognormal(in), lognormal(out)."""
    rng = np.random.default_rng(seed)
    peak = spec.peak_rate
    mu_in, mu_out = math.log(spec.input_len_median), math.log(spec.output_len_median)
    out = []
    t = 0.0
    while True:
        t += rng.exponential(1.0 / peak)
        if t >= spec.duration:
            return out
        if rng.uniform() * peak > spec.rate_at(t):
            continue
        li = max(1, int(rng.lognormal(mu_in, spec.input_len_sigma)))
        lo = max(0, int(rng.lognormal(mu_out, spec.output_len_sigma)))
        out.append(RequestRecord(t, li, lo))


def tail_length(lengths, q: float) -> int:
    """'higher' empirical quantile: smallest value covering q."""
    ordered = sorted(lengths)
    return ordered[max(0, math.ceil(q * len(ordered)) - 1)]


def windowize(records, window_len: float = 60.0, quantile: float = 0.95):
    """[(prefill, decode)] WorkloadPoints per window. Prefill: arrivals/s at
    the q-tail input length; decode: generated tokens/s at length 1; empty
    windows give qps = 0 points."""
    if window_len <= 0:
        raise ValueError("window_len must be positive")
    if not (0.0 < quantile <= 1.0):
        raise ValueError("quantile must be in (0, 1]")
    if not records:
        return []
    horizon = max(r.arrival_time for r in records)
    n = max(1, math.ceil(horizon / window_len + 1e-12))
    buckets = [[] for _ in range(n)]
    for r in records:
        buckets[min(int(r.arrival_time / window_len), n - 1)].append(r)
    result = []
    for i, bucket in enumerate(buckets):
        win = (i * window_len, (i + 1) * window_len)
        if bucket:
            pre = WorkloadPoint(len(bucket) / window_len,
                                max(1, tail_length([r.input_len for r in bucket], quantile)),
                                "prefill", win)
            dec = WorkloadPoint(sum(r.output_len for r in bucket) / window_len, 1, "decode", win)
        else:
            pre = WorkloadPoint(0.0, 1, "prefill", win)
            dec = WorkloadPoint(0.0, 1, "decode", win)
        result.append((pre, dec))
    return result


def windowize_device(arrival, input_len, output_len, window_len: float = 60.0,
                     quantile: float = 0.95, device="cuda", max_windows=None):
    """windowize on the GPU (opsc_windowize, csrc/k_windowize.cu). Inputs are
    record arrays (host or device); returns device tensors (prefill_qps,
    prefill_len, decode_qps) of length n_windows, already resident in HBM for
    the planners."""
    import ctypes as C

    import torch

    from . import _native, abi
    if window_len <= 0:
        raise ValueError("window_len must be positive")
    if not (0.0 < quantile <= 1.0):
        raise ValueError("quantile must be in (0, 1]")
    dev = torch.device(device)
    t = torch.as_tensor(arrival, dtype=torch.float64, device=dev).contiguous()
    li = torch.as_tensor(input_len, dtype=torch.int32, device=dev).contiguous()
    lo = torch.as_tensor(output_len, dtype=torch.int32, device=dev).contiguous()
    n = int(t.numel())
    if n == 0:
        z = torch.zeros(0, dtype=torch.float64, device=dev)
        return z, torch.zeros(0, dtype=torch.int32, device=dev), z
    if max_windows is None:
        horizon = float(t.max().item())
        max_windows = max(1, math.ceil(horizon / window_len + 1e-12))
    L = _native.load()
    ws_bytes = L.opsc_windowize_workspace(n, max_windows)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
    nw = torch.zeros(1, dtype=torch.int32, device=dev)
    pq = torch.empty(max_windows, dtype=torch.float64, device=dev)
    pl = torch.empty(max_windows, dtype=torch.int32, device=dev)
    dq = torch.empty(max_windows, dtype=torch.float64, device=dev)
    rec = abi.OpscTraceRecords(n, t.data_ptr(), li.data_ptr(), lo.data_ptr())
    _native.check(L.opsc_windowize(rec, float(window_len), float(quantile), max_windows,
                                   nw.data_ptr(), pq.data_ptr(), pl.data_ptr(), dq.data_ptr(),
                                   ws.data_ptr(), C.c_size_t(ws_bytes),
                                   torch.cuda.current_stream(dev).cuda_stream), "opsc_windowize")
    k = int(nw.item())
    if k > max_windows:
        raise ValueError(f"trace spans {k} windows > max_windows={max_windows}")
    return pq[:k], pl[:k], dq[:k]


def windowize_points(records, window_len: float = 60.0, quantile: float = 0.95, device="cuda"):
    """Drop-in for windowize() computed on the GPU: [(prefill, decode)] points."""
    if window_len <= 0:
        raise ValueError("window_len must be positive")
    if not (0.0 < quantile <= 1.0):
        raise ValueError("quantile must be in (0, 1]")
    if not records:
        return []
    arr = np.array([r.arrival_time for r in records], dtype=np.float64)
    li = np.array([r.input_len for r in records], dtype=np.int32)
    lo = np.array([r.output_len for r in records], dtype=np.int32)
    pq, pl, dq = (x.cpu().numpy() for x in windowize_device(arr, li, lo, window_len, quantile, device))
    out = []
    for i in range(len(pq)):
        win = (i * window_len, (i + 1) * window_len)
        out.append((WorkloadPoint(float(pq[i]), int(pl[i]), "prefill", win),
                    WorkloadPoint(float(dq[i]), 1, "decode", win)))
    return out
