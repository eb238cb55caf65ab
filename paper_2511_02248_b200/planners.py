"""Drop-in planners: the reference's planner signatures, searched on the GPU.

  brute_force_autoscale(dag, profiles, point, params, bounds=None)
      autoscaler.py:706-847 -- exhaustive (P,R,B)^n argmin, on device
  model_level_autoscale(dag, profiles, point, params)
      autoscaler.py:596-681 -- uniform (B,R) probe/bisect, on device
  plan_windows(dag, profiles, points, params, mode, bounds=None)
      batched form of the above over many WorkloadPoints (new; equals mapping
      the per-point call over `points`, minus the per-point launch cost)

Argument checks and exceptions follow the reference in its order:
ValueError for qps <= 0 and UnknownProfile (_Evaluator, :148-150), the >6-op
and MAX_ENUMERATION guards (:725-738; MAX_ENUMERATION is read at call time,
so patching it works as in the reference), UnknownPhase (first predict_op),
then the device-reported NoStableConfig cases (:289, :835, :678).

The batched entry lifts the 6-op / MAX_ENUMERATION guards by default (it is
the path for the 10-op 70B DAG and ~1e8-candidate windows); the per-point
planners keep them unless called with guards=False.
"""

from __future__ import annotations

import math
import threading
from operator import is_

import numpy as np
from collections import OrderedDict

from . import _native, abi, errors, model, tables
from .plans import WindowDecisions

MAX_ENUMERATION = 10_000_000
MAX_BRUTE_FORCE_OPS = 6


class _Packed:
    """LRU of packed tables for the per-point API.

    The reference's planners are called once per WorkloadPoint with the same
    DAG / ProfileSet / AutoscaleParams objects (runner.run_point,
    cli.cmd_autoscale's window loop), and repacking them dominated the
    per-point cost. Entries are keyed by object identity and hold strong
    references, so an id cannot be reused while cached; a ProfileSet (a
    mutable container in the reference, perfmodel.py:111-130) is revalidated
    by a cheap signature of its contents' identities, link bandwidth and
    interference model. OperatorDag and AutoscaleParams / BruteForceBounds are
    immutable by the reference's contract (opgraph.py:71-76, frozen
    dataclasses at autoscaler.py:102, 688)."""

    def __init__(self, size=32):
        self.size, self.lock, self.d = size, threading.Lock(), OrderedDict()

    def get(self, key, refs, sig, make):
        with self.lock:
            hit = self.d.get(key)
            if hit is not None and hit[1] == sig and all(map(is_, hit[0], refs)):
                self.d.move_to_end(key)
                return hit[2]
        val = make()
        with self.lock:
            self.d[key] = (refs, sig, val)
            while len(self.d) > self.size:
                self.d.popitem(last=False)
        return val


_PROBLEMS, _SPECS = _Packed(), _Packed(128)


def _profile_sig(dag, profiles):
    profs = getattr(profiles, "profiles", None)
    return (len(dag.nodes), len(dag.edges), getattr(profiles, "link_bandwidth", None),
            id(getattr(profiles, "interference", None)), id(profs),
            tuple(map(id, profs.values())) if isinstance(profs, dict) else None)


def packed_problem(dag, profiles):
    """tables.pack_problem, cached per (DAG, ProfileSet) object."""
    return _PROBLEMS.get((id(dag), id(profiles)), (dag, profiles), _profile_sig(dag, profiles),
                         lambda: tables.pack_problem(dag, profiles))


def _spec(kind, problem, params, bounds, make):
    return _SPECS.get((kind, id(problem), id(params), id(bounds)), (problem, params, bounds), None, make)


def _guard(problem, params, bounds, max_enumeration, err):
    ops = problem.ids
    if len(ops) > MAX_BRUTE_FORCE_OPS:
        raise err.SearchSpaceTooLarge(f"{len(ops)} operators > {MAX_BRUTE_FORCE_OPS}")
    projected = 1
    for op in ops:
        projected *= (len(bounds.parallelism_for(params, op)) * bounds.b_max_for(params, op)
                      * bounds.r_max)
    if projected > max_enumeration:
        raise err.SearchSpaceTooLarge(
            f"projected enumeration {projected} exceeds {max_enumeration}")


def _points_ok(points):
    for p in points:
        if p.qps <= 0:  # autoscaler.py:148-149 (NaN passes; see plans.nonfinite_qps)
            raise ValueError("workload point must have qps > 0")


def brute_force_autoscale(dag, profiles, point, params, bounds=None, *, guards=True,
                          fleet=None, energy=None, types=model, err=errors,
                          max_enumeration=None):
    """Exact minimum-objective plan over the bounded configuration space
    (ties: lexicographically smallest config vector in node-id order)."""
    bounds = bounds if bounds is not None else types.BruteForceBounds()
    _points_ok([point])
    problem = packed_problem(dag, profiles)
    if guards:
        _guard(problem, params, bounds,
               MAX_ENUMERATION if max_enumeration is None else max_enumeration, err)
    return _run(abi.MODE_ORACLE, problem, [point], params, bounds, fleet, energy, types, err,
                single=True).plan(0)


def model_level_autoscale(dag, profiles, point, params, *, fleet=None, energy=None,
                          types=model, err=errors):
    """Monolithic baseline: one (B, R) shared by every operator."""
    _points_ok([point])
    problem = packed_problem(dag, profiles)
    return _run(abi.MODE_MODEL, problem, [point], params, None, fleet, energy, types, err,
                single=True).plan(0)


def greedy_autoscale(dag, profiles, point, params, *, fleet=None, energy=None, types=model,
                     err=errors, trace_cap=4096):
    """Greedy bottleneck-driven operator-level planner (Alg. 1 as the reference
    codes it, autoscaler.py:334-589), one CTA per window on the device; the
    returned plan carries the reference's move trace."""
    _points_ok([point])
    problem = packed_problem(dag, profiles)
    return _run(abi.MODE_OPERATOR, problem, [point], params, None, fleet, energy, types, err,
                trace_cap, single=True).plan(0)


_TLS = threading.local()


def _single_io(point, params, n_ops, tcap):
    """Per-thread W=1 window / decision buffers of the per-point planners
    (their plan is materialised before the call returns, so the next call may
    overwrite them)."""
    io = getattr(_TLS, "io", None)
    if io is None:
        io = _TLS.io = {}
    win = io.get("win")
    if win is None:
        win = io["win"] = tables.WindowArrays(np.zeros(1), np.zeros(1, np.int32), np.zeros(1, np.uint8),
                                              np.zeros(1), np.zeros(1))
    win.qps[0], win.seq_len[0] = point.qps, point.seq_len
    win.phase[0] = tables.PHASE_INDEX[point.phase]
    win.slo[0], win.eps[0] = params.slo, params.epsilon
    out = io.get((n_ops, tcap))
    if out is None:
        out = io[(n_ops, tcap)] = tables.DecisionArrays(1, n_ops, tcap)
    return win, out


def _run(mode, problem, points, params, bounds, fleet, energy, types, err, trace_cap=4096, single=False,
         certify=False):
    phases = {p.phase for p in points}
    for ph in sorted(phases):
        problem.require_phase(ph)
    out = None
    if single:
        win, out = _single_io(points[0], params, problem.n_ops,
                              trace_cap if mode == abi.MODE_OPERATOR else 0)
    else:
        win = tables.pack_windows(points, params.slo, params.epsilon)
    grid = spec = greedy = None
    if mode == abi.MODE_ORACLE:
        grid = _spec("grid", problem, params, bounds, lambda: tables.pack_grid(problem, params, bounds))
    elif mode == abi.MODE_MODEL:
        spec = _spec("model", problem, params, None, lambda: tables.pack_model(problem, params))
    else:
        greedy = _spec("greedy", problem, params, None, lambda: tables.pack_greedy(problem, params))
    place = _SPECS.get(("place", id(fleet), id(energy)), (fleet, energy),
                       None if fleet is None else tuple(map(id, fleet)),
                       lambda: tables.pack_place(fleet, energy))
    arrays = _native.plan_windows_host(mode, problem, win, grid=grid, model=spec, place=place,
                                       greedy=greedy, trace_cap=trace_cap, out=out, certify=certify)
    return WindowDecisions(problem, points, arrays, mode, types, err, r_cap=params.r_cap)


_MODES = {"oracle": abi.MODE_ORACLE, "model": abi.MODE_MODEL, "operator": abi.MODE_OPERATOR}


def decide_windows(dag, profiles, points, params, mode="oracle", bounds=None, *,
                   fleet=None, energy=None, guards=False, types=model, err=errors, certify=False):
    """Batched planning over many WorkloadPoints.

    `params` is an AutoscaleParams or a {phase: AutoscaleParams} map (prefill
    SLO = TTFT, decode SLO = TBT; cli.py:114-120). Points with qps <= 0 are
    idle windows: they get no plan (cli.py:138-144). Returns a list of
    WindowDecisions groups aligned with `points` via .index.

    certify=True (brute force only) also runs the summation-order
    certificate: WindowDecisions.order_sensitive(k) is True for windows whose
    decision could differ under the reference's frozenset-ordered leaf sum
    (autoscaler.py:792-796), i.e. where some candidate that could win lies
    within 64 ulps of the SLO. The decisions themselves are unchanged.
    """
    m = _MODES[mode] if isinstance(mode, str) else mode
    bounds = bounds if (bounds is not None or m != abi.MODE_ORACLE) else types.BruteForceBounds()
    problem = packed_problem(dag, profiles)
    by_phase = params if isinstance(params, dict) else None
    groups = {}
    for i, p in enumerate(points):
        if p.qps <= 0:  # idle window (cli.py:138)
            continue
        groups.setdefault(p.phase, []).append(i)
    out = []
    for ph, idx in sorted(groups.items()):
        prm = by_phase[ph] if by_phase is not None else params
        if guards and m == abi.MODE_ORACLE:
            _guard(problem, prm, bounds, MAX_ENUMERATION, err)
        dec = _run(m, problem, [points[i] for i in idx], prm, bounds, fleet, energy, types, err,
                   certify=certify)
        dec.index = idx
        out.append(dec)
    return out


def plan_windows(dag, profiles, points, params, mode="oracle", bounds=None, *, fleet=None,
                 energy=None, guards=False, types=model, err=errors):
    """list[ScalingPlan | None] aligned with `points` (None for idle windows).
    Errors of individual windows raise, as the per-point call would."""
    plans = [None] * len(points)
    for dec in decide_windows(dag, profiles, points, params, mode, bounds, fleet=fleet,
                              energy=energy, guards=guards, types=types, err=err):
        for k, i in enumerate(dec.index):
            plans[i] = dec.plan(k)
    return plans


def candidate_space(problem, grid):
    """Semantic candidate count (|P|*R*B)^n of one window."""
    return math.prod(tables.menu_sizes(problem, grid))
