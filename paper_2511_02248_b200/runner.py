"""Batched scenario runner: plan, place and score many workload points per
launch, with the reference runner's results and byte-identical artifacts.

The reference (runner.py:55-173, 190-284; cli.py:123-217) plans and places
one point at a time -- a Python call chain per window and per sweep value.
Here every point of a trace or sweep that shares a DAG goes to the device in
one planning launch (K1-K5, one CTA/thread group per window) and one
placement launch (K6, CTA per window, per-window SLO, shared or
default-stream), and only the host-side object and text assembly remains:

  evaluate_points  -- run_point over many points (plan + place + ScenarioEval)
  compare_points   -- compare_point over many points
  sweep            -- runner.sweep, one batch per axis (model_scale: per value)
  sweep_rows_to_csv, fmt, workload_fingerprint, compare -- the reference's
                      deterministic formats, restated
  autoscale_windows -- cli.cmd_autoscale's artifacts (plan_*.json,
                      placement_*.json, metrics.csv) from a windowed trace

Errors keep the reference's order: outcomes are computed for the whole batch,
then consumed in the reference's loop order, so the first exception the
reference would raise is the one raised, after the same files were written.
"""

from __future__ import annotations

import hashlib
import json
import math
from dataclasses import dataclass, replace
from pathlib import Path

import numpy as np

from . import _native, abi, errors, model, placement as plc, planners, tables
from .plans import WindowDecisions

MODES = ("operator", "model", "oracle")
PLACEMENTS = ("shared", "default_stream")
_MODE_CODE = {"operator": abi.MODE_OPERATOR, "model": abi.MODE_MODEL, "oracle": abi.MODE_ORACLE}


# --------------------------------------------------------------------------
# result types (runner.py:28-35, 108-141; metrics.py:50-81)


@dataclass
class PointResult:
    point: object
    mode: str
    placement_mode: str
    plan: object
    placement: object
    evaluation: object


@dataclass(frozen=True)
class ScenarioEval:
    label: str
    fingerprint: str
    devices_used: int
    energy_joules: float
    memory_bytes: float
    feasible: bool


@dataclass
class SavingsReport:
    gpu_savings: float
    energy_savings: float
    memory_savings: float
    baseline_label: str
    candidate_label: str
    baseline: dict
    candidate: dict

    def to_dict(self) -> dict:
        return {
            "gpu_savings": self.gpu_savings,
            "energy_savings": self.energy_savings,
            "memory_savings": self.memory_savings,
            "baseline_label": self.baseline_label,
            "candidate_label": self.candidate_label,
            "baseline": self.baseline,
            "candidate": self.candidate,
        }


@dataclass
class ComparisonRow:
    axis: str
    value: float
    point: object
    baseline: object
    candidate: object
    report: object

    @property
    def vacuous(self) -> bool:
        return self.baseline is None and self.candidate is None

    @property
    def feasible_baseline(self) -> bool:
        return self.vacuous or (self.baseline is not None and self.baseline.evaluation.feasible)

    @property
    def feasible_candidate(self) -> bool:
        return self.vacuous or (self.candidate is not None and self.candidate.evaluation.feasible)

    @property
    def fingerprint(self) -> str:
        for side in (self.baseline, self.candidate):
            if side is not None:
                return side.evaluation.fingerprint
        return ""


class Types:
    """Constructors the runner emits; `installer` swaps in the reference's."""

    PointResult = PointResult
    ScenarioEval = ScenarioEval
    SavingsReport = SavingsReport
    ComparisonRow = ComparisonRow
    plan_types = model
    err = errors


# --------------------------------------------------------------------------
# deterministic formats (metrics.py:135-147, 150-190; runner.py:243-284)


def workload_fingerprint(point, slo, extra=None) -> str:
    """sha256 prefix of the sorted-key JSON of the point and SLO."""
    payload = {"qps": point.qps, "seq_len": point.seq_len, "phase": point.phase,
               "window": list(point.window), "slo": slo}
    if extra:
        payload.update(extra)
    return hashlib.sha256(json.dumps(payload, sort_keys=True).encode()).hexdigest()[:16]


def compare(baseline, candidate, T=Types):
    """Savings fractions of candidate over baseline (unclamped)."""
    if baseline.fingerprint != candidate.fingerprint:
        raise T.err.MismatchedScenario(
            f"fingerprints differ: {baseline.fingerprint} vs {candidate.fingerprint}")
    for name, value in (("devices_used", baseline.devices_used),
                        ("energy_joules", baseline.energy_joules),
                        ("memory_bytes", baseline.memory_bytes)):
        if value <= 0:
            raise ValueError(f"baseline {name} must be positive, got {value}")
    side = lambda e: {"devices": e.devices_used, "energy_joules": e.energy_joules,
                      "memory_bytes": e.memory_bytes, "feasible": e.feasible}
    return T.SavingsReport(
        gpu_savings=(baseline.devices_used - candidate.devices_used) / baseline.devices_used,
        energy_savings=(baseline.energy_joules - candidate.energy_joules) / baseline.energy_joules,
        memory_savings=(baseline.memory_bytes - candidate.memory_bytes) / baseline.memory_bytes,
        baseline_label=baseline.label, candidate_label=candidate.label,
        baseline=side(baseline), candidate=side(candidate))


def fmt(x: float) -> str:
    if x != x:
        return ""
    if math.isinf(x):
        return "inf" if x > 0 else "-inf"
    return f"{x:.10g}"


SWEEP_CSV_HEADER = ("sweep_var,value,gpu_savings,energy_savings,memory_savings,"
                    "feasible_baseline,feasible_candidate,fingerprint")

METRICS_CSV_HEADER = ("window_start,window_end,phase,qps,seq_len,mode,placement,feasible,"
                      "devices,energy_joules,memory_bytes,plan_latency,placed_latency,"
                      "objective,fingerprint")


def sweep_rows_to_csv(rows) -> str:
    lines = [SWEEP_CSV_HEADER]
    for row in rows:
        if row.report is not None:
            g, e, m = (fmt(row.report.gpu_savings), fmt(row.report.energy_savings),
                       fmt(row.report.memory_savings))
        elif row.vacuous:
            g = e = m = fmt(0.0)
        else:
            g = e = m = ""
        lines.append(",".join([row.axis, fmt(row.value), g, e, m, str(row.feasible_baseline).lower(),
                               str(row.feasible_candidate).lower(), row.fingerprint]))
    return "\n".join(lines) + "\n"


# --------------------------------------------------------------------------
# batched run_point


class _Raise:
    """An outcome that raises when consumed (the reference raised there)."""

    def __init__(self, exc):
        self.exc = exc


def _plan_key(params):
    # points whose params differ only in slo / epsilon share one launch
    # (slo and epsilon travel per window in OpscWindows)
    return repr(replace(params, slo=1.0, epsilon=0.0))


def _plan_batch(mode, dag, profiles, points, params_list, bounds, T, max_enumeration):
    """(plans or _Raise per point, packed problem or None) for points with
    qps > 0, one launch per params group."""
    m = _MODE_CODE.get(mode)
    out = [None] * len(points)
    if m is None:
        return [_Raise(ValueError(f"unknown mode {mode!r}"))] * len(points), None
    try:
        problem = tables.pack_problem(dag, profiles)
    except Exception as exc:  # UnknownProfile etc.: every point raises it
        return [_Raise(exc)] * len(points), None
    PT, E = T.plan_types, T.err
    if m == abi.MODE_ORACLE and bounds is None:
        bounds = PT.BruteForceBounds()
    groups = {}
    for i, prm in enumerate(params_list):
        groups.setdefault(_plan_key(prm), []).append(i)
    for idx in groups.values():
        prm = params_list[idx[0]]
        try:
            # brute_force_autoscale's order: guards, then the phase lookup
            if m == abi.MODE_ORACLE:
                planners._guard(problem, prm, bounds, planners.MAX_ENUMERATION if max_enumeration is None
                                else max_enumeration, E)
            for ph in sorted({points[i].phase for i in idx}):
                problem.require_phase(ph)
            pts = [points[i] for i in idx]
            win = tables.pack_windows(pts, [params_list[i].slo for i in idx],
                                      [params_list[i].epsilon for i in idx])
            grid = tables.pack_grid(problem, prm, bounds) if m == abi.MODE_ORACLE else None
            spec = tables.pack_model(problem, prm)
            greedy = tables.pack_greedy(problem, prm) if m == abi.MODE_OPERATOR else None
            arrays = _native.plan_windows_host(m, problem, win, grid=grid, model=spec,
                                               place=tables.pack_place(), greedy=greedy)
            dec = WindowDecisions(problem, pts, arrays, m, PT, E, r_cap=prm.r_cap)
        except Exception as exc:
            for i in idx:
                out[i] = _Raise(exc)
            continue
        for k, i in enumerate(idx):
            try:
                out[i] = dec.plan(k)
            except Exception as exc:
                out[i] = _Raise(exc)
    return out, problem


def evaluate_points(mode, dag, profiles, fleet, points, params, placement_mode="shared",
                    energy_params=None, bounds=None, fingerprint_extra=None, *, types=Types,
                    max_enumeration=None):
    """runner.run_point (runner.py:55-105) for many points of one DAG.

    `params` is one AutoscaleParams or a list aligned with `points`;
    `fingerprint_extra` likewise. Returns a list aligned with `points` of
    PointResult or _Raise (consume with `result()`); points must have qps > 0.
    """
    T = types
    n = len(points)
    params_list = params if isinstance(params, (list, tuple)) else [params] * n
    extras = (fingerprint_extra if isinstance(fingerprint_extra, (list, tuple))
              else [fingerprint_extra] * n)
    energy_params = energy_params or model.EnergyParams()
    plans, problem = _plan_batch(mode, dag, profiles, points, params_list, bounds, T, max_enumeration)
    if problem is None:  # every point failed before packing
        return plans
    label = f"{mode}/{placement_mode}"
    results = [None] * n
    to_place = []
    for i, plan in enumerate(plans):
        if isinstance(plan, _Raise):
            results[i] = plan
            continue
        fp = workload_fingerprint(points[i], params_list[i].slo, extras[i])
        if not plan.feasible:
            ev = T.ScenarioEval(label=label, fingerprint=fp, devices_used=0, energy_joules=0.0,
                                memory_bytes=0.0, feasible=False)
            results[i] = T.PointResult(points[i], mode, placement_mode, plan, None, ev)
        elif placement_mode not in PLACEMENTS:
            results[i] = _Raise(ValueError(f"unknown placement mode {placement_mode!r}"))
        elif not fleet:
            results[i] = _Raise(ValueError("fleet must not be empty"))
        else:
            to_place.append((i, fp))
    if not to_place:
        return results
    idx = [i for i, _ in to_place]
    cfg = np.zeros((len(idx), problem.n_ops, 3), np.int16)
    for k, i in enumerate(idx):
        for op, c in plans[i].configs.items():
            cfg[k, problem.rank[op]] = (c.p, c.r, c.b)
    win = tables.pack_windows([points[i] for i in idx], [params_list[i].slo for i in idx], 0.0)
    sf = plc.SharedFleet.from_params(fleet, model.PlacementParams(slo=params_list[idx[0]].slo),
                                     profiles, energy_params,
                                     default_stream=placement_mode == "default_stream",
                                     window_slo=True)
    # brute force builds configs in sorted-id order, the other planners in
    # dag.node_ids order (the energy sum follows plan.configs order)
    order = 0 if mode == "oracle" else 1
    arr = plc.place_windows(problem, win, cfg, np.ones(len(idx), np.uint8), sf, order)
    for k, (i, fp) in enumerate(to_place):
        try:
            plc.raise_placement_status(int(arr.status[k]), len(fleet), T.err)
        except Exception as exc:
            results[i] = _Raise(exc)
            continue
        plan = plans[i]
        placed = plc.placement_object(arr, k, plan, dag, profiles, problem, sf, points[i].seq_len,
                                      T.plan_types)
        ev = T.ScenarioEval(label=label, fingerprint=fp, devices_used=placed.devices_used,
                            energy_joules=float(arr.energy[k]), memory_bytes=float(arr.memory[k]),
                            feasible=plan.feasible and placed.feasible)
        results[i] = T.PointResult(points[i], mode, placement_mode, plan, placed, ev)
    return results


def result(outcome):
    """PointResult of an evaluate_points outcome, raising the reference's error."""
    if isinstance(outcome, _Raise):
        raise outcome.exc
    return outcome


def run_point(mode, dag, profiles, fleet, point, params, placement_mode="shared",
              energy_params=None, bounds=None, fingerprint_extra=None, *, types=Types):
    """Drop-in for runner.run_point (one point)."""
    return result(evaluate_points(mode, dag, profiles, fleet, [point], params, placement_mode,
                                  energy_params, bounds, fingerprint_extra, types=types)[0])


# --------------------------------------------------------------------------
# comparisons and sweeps


def compare_points(dag, profiles, fleet, points, params, placement_mode="shared",
                   energy_params=None, axis="", values=None, fingerprint_extra=None, *,
                   types=Types):
    """compare_point (runner.py:144-173) for many points of one DAG: one
    batched model-level baseline (shared placement) and one batched
    operator-level candidate. Returns outcomes (ComparisonRow or _Raise)."""
    T = types
    n = len(points)
    params_list = params if isinstance(params, (list, tuple)) else [params] * n
    extras = (fingerprint_extra if isinstance(fingerprint_extra, (list, tuple))
              else [fingerprint_extra] * n)
    values = values if values is not None else [0.0] * n
    # the reference's predicate: vacuous iff qps <= 0.0 (runner.py:157); NaN is live
    live = [i for i in range(n) if not isinstance(points[i], _Raise) and not points[i].qps <= 0.0]
    sub = lambda seq: [seq[i] for i in live]
    base = evaluate_points("model", dag, profiles, fleet, sub(points), sub(params_list), "shared",
                           energy_params, None, sub(extras), types=T) if live else []
    cand = evaluate_points("operator", dag, profiles, fleet, sub(points), sub(params_list),
                           placement_mode, energy_params, None, sub(extras), types=T) if live else []
    out = [None] * n
    for i in range(n):
        if isinstance(points[i], _Raise):
            out[i] = points[i]
        elif points[i].qps <= 0.0:
            out[i] = T.ComparisonRow(axis, values[i], points[i], None, None, None)
    for k, i in enumerate(live):
        b, c = base[k], cand[k]
        if isinstance(b, _Raise):
            out[i] = b
            continue
        if isinstance(c, _Raise):
            out[i] = c
            continue
        try:
            rep = (compare(b.evaluation, c.evaluation, T)
                   if b.evaluation.feasible and c.evaluation.feasible else None)
        except Exception as exc:
            out[i] = _Raise(exc)
            continue
        out[i] = T.ComparisonRow(axis, values[i], points[i], b, c, rep)
    return out


def scale_dag(dag, factor):
    """Model-size sweep: every node's layer repeat count scaled (runner.py:176-187)."""
    N = type(dag.nodes[0]) if dag.nodes else model.OperatorNode
    nodes = [N(id=n.id, kind=n.kind, layer_count=max(1, round(n.layer_count * factor)),
               profile_ref=n.profile_ref) for n in dag.nodes]
    return type(dag)(nodes=nodes, edges=list(dag.edges))


def sweep(axis, values, dag, profiles, fleet, base_point, params, placement_mode="shared",
          energy_params=None, max_workers=4, *, types=Types):
    """runner.sweep (runner.py:190-240): rows in axis order; seqlen and qps
    run as one batch per side, model_scale as one launch pair per value.
    `max_workers` is accepted for signature parity (the batch replaces the
    thread pool)."""
    del max_workers
    if axis not in ("seqlen", "qps", "model_scale"):
        raise ValueError(f"unknown sweep axis {axis!r}")
    T = types
    extras = [{"axis": axis, "value": v} for v in values]
    if axis == "model_scale":
        rows = []
        for v, ex in zip(values, extras):
            rows += compare_points(scale_dag(dag, v), profiles, fleet, [base_point], [params],
                                   placement_mode, energy_params, axis, [v], [ex], types=T)
    else:
        points, prms = [], []
        for v in values:
            try:
                if axis == "seqlen":
                    # offered token load and SLO pressure held constant (runner.py:215-225)
                    scale = v / base_point.seq_len
                    points.append(replace(base_point, seq_len=int(v), qps=base_point.qps / scale))
                    prms.append(replace(params, slo=params.slo * scale, epsilon=params.epsilon * scale))
                else:
                    points.append(replace(base_point, qps=float(v)))
                    prms.append(params)
            except Exception as exc:
                points.append(_Raise(exc))
                prms.append(params)
        rows = compare_points(dag, profiles, fleet, points, prms, placement_mode, energy_params,
                              axis, list(values), extras, types=T)
    return [result(r) for r in rows]


# --------------------------------------------------------------------------
# cli.cmd_autoscale artifacts


def autoscale_windows(dag, profiles, fleet, windows, mode, placement_mode, params_for_phase, out_dir,
                      *, types=Types, bounds=None, max_enumeration=None):
    """cli.cmd_autoscale (cli.py:123-186) over windowed (prefill, decode)
    points: writes plan_NNN_<phase>.json / placement_NNN_<phase>.json and
    metrics.csv with the reference's bytes; returns the exit code (0, or 2
    if some point is infeasible). `params_for_phase(phase)` builds the
    AutoscaleParams (and may raise, as cli._params does)."""
    out = Path(out_dir)
    out.mkdir(parents=True, exist_ok=True)
    prm = {}
    for ph in ("prefill", "decode"):
        try:
            prm[ph] = params_for_phase(ph)
        except Exception as exc:
            prm[ph] = _Raise(exc)
    live = [(i, pt) for i, pair in enumerate(windows) for pt in pair
            if not pt.qps <= 0.0 and not isinstance(prm[pt.phase], _Raise)]  # cli.py:138
    res = {}
    if live:
        outcomes = evaluate_points(mode, dag, profiles, fleet, [pt for _, pt in live],
                                   [prm[pt.phase] for _, pt in live], placement_mode,
                                   bounds=bounds, types=types, max_enumeration=max_enumeration)
        res = {(i, pt.phase): o for (i, pt), o in zip(live, outcomes)}
    rows = [METRICS_CSV_HEADER]
    any_infeasible = False
    for i, (prefill, decode) in enumerate(windows):
        for point in (prefill, decode):
            tag = f"{i:03d}_{point.phase}"
            if point.qps <= 0.0:
                rows.append(f"{fmt(point.window[0])},{fmt(point.window[1])},"
                            f"{point.phase},0,1,{mode},{placement_mode},true,0,0,0,0,0,0,")
                continue
            if isinstance(prm[point.phase], _Raise):
                raise prm[point.phase].exc
            r = result(res[(i, point.phase)])
            (out / f"plan_{tag}.json").write_text(
                json.dumps(r.plan.to_dict(), indent=2, sort_keys=True) + "\n")
            if r.placement is not None:
                (out / f"placement_{tag}.json").write_text(
                    json.dumps(r.placement.to_dict(), indent=2, sort_keys=True) + "\n")
            ev = r.evaluation
            if not ev.feasible:
                any_infeasible = True
            placed_latency = r.placement.recomputed_latency if r.placement else ""
            rows.append(",".join([
                fmt(point.window[0]), fmt(point.window[1]), point.phase, fmt(point.qps),
                str(point.seq_len), mode, placement_mode, str(ev.feasible).lower(),
                str(ev.devices_used), fmt(ev.energy_joules), fmt(ev.memory_bytes),
                fmt(r.plan.iteration_latency), fmt(placed_latency) if placed_latency != "" else "",
                str(r.plan.objective), ev.fingerprint]))
    (out / "metrics.csv").write_text("\n".join(rows) + "\n")
    return 2 if any_infeasible else 0
