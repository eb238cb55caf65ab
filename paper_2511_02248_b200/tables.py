"""Pack planner inputs into the C-ABI tables of include/opscale_b200.h.

Everything here runs once per planning instance on the host and only reads
the reference-shaped objects (duck typing: the reference's own OperatorDag /
ProfileSet / AutoscaleParams / BruteForceBounds / WorkloadPoint work as well
as this package's mirrors):

  * operators are re-indexed by their rank in sorted(node_ids), which is the
    brute-force lexicographic order (autoscaler.py:725);
  * topological order, predecessor sets and sinks come from the DAG
    (opgraph.py:71-148);
  * out-edge volume profiles are listed in dag.out_edges order
    (autoscaler.py:163-172);
  * menus follow BruteForceBounds (autoscaler.py:688-700, 747-749).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

from operator import is_

import numpy as np

from . import abi
from .errors import UnknownPhase

PHASE_INDEX = {"prefill": 0, "decode": 1}


@dataclass
class Problem:
    """A DAG + ProfileSet packed as an OpscDag, with the id <-> rank maps."""

    dag: object
    profiles: object
    ids: list            # lex rank -> op id
    rank: dict           # op id -> lex rank
    table: abi.OpscDag

    @property
    def n_ops(self):
        return len(self.ids)

    @property
    def node_order(self):
        """Lex ranks in dag.node_ids order (the model level's / greedy's config order)."""
        return [self.table.node_order[k] for k in range(len(self.ids))]

    def require_phase(self, phase):
        """UnknownPhase exactly when some operator's profile lacks `phase`
        (perfmodel.py:100-105), which the reference hits on the first
        predict_op of that operator."""
        if phase not in PHASE_INDEX:
            raise UnknownPhase(f"unknown phase {phase!r}")
        bit = self.table.has_phase[PHASE_INDEX[phase]]
        for v, op in enumerate(self.ids):
            if not (bit >> v) & 1:
                prof = self.profiles.get(self.dag.node(op).profile_ref)
                prof.latency_model(phase)  # raises the profile's own UnknownPhase
                raise UnknownPhase(f"profile {prof.name} has no {phase} model")


def pack_problem(dag, profiles) -> Problem:
    profiles.validate_against(dag)  # UnknownProfile, as _Evaluator does (autoscaler.py:150)
    ids = sorted(dag.node_ids)
    n = len(ids)
    if n > abi.MAX_OPS:
        raise ValueError(f"{n} operators exceed the {abi.MAX_OPS}-operator table limit")
    rank = {op: i for i, op in enumerate(ids)}
    t = abi.OpscDag()
    t.n_ops = n
    for i, op in enumerate(dag.topo_order):
        t.topo[i] = rank[op]
    for i, op in enumerate(dag.node_ids):
        t.node_order[i] = rank[op]
    edge_i = 0
    sink = 0
    has = [0, 0]
    for v, op in enumerate(ids):
        node = dag.node(op)
        prof = profiles.get(node.profile_ref)
        t.layer_count[v] = int(node.layer_count)
        mask = 0
        for p in dag.predecessors(op):
            mask |= 1 << rank[p]
        t.pred_mask[v] = mask
        if not dag.successors(op):
            sink |= 1 << v
        for ph, k in PHASE_INDEX.items():
            model = prof.phase_models.get(ph)
            if model is not None:
                has[k] |= 1 << v
                t.c0[k][v], t.c1[k][v], t.c2[k][v] = float(model.c0), float(model.c1), float(model.c2)
        t.eta[v] = float(prof.eta)
        t.weight_mem[v] = float(prof.weight_mem)
        t.m0[v], t.m1[v] = float(prof.m0), float(prof.m1)
        t.s0[v], t.s1[v] = float(prof.s0), float(prof.s1)
        t.out_ptr[v] = edge_i
        for e in dag.out_edges(op):
            if edge_i >= abi.MAX_EDGES:
                raise ValueError(f"more than {abi.MAX_EDGES} edges")
            vp = profiles.get(e.volume_ref)
            t.out_v0[edge_i], t.out_v1[edge_i] = float(vp.v0), float(vp.v1)
            edge_i += 1
    t.out_ptr[n] = edge_i
    t.n_edges = edge_i
    t.sink_mask = sink
    t.has_phase[0], t.has_phase[1] = has
    bw = float(profiles.link_bandwidth)
    if bw <= 0.0:
        raise ValueError(f"bandwidth must be positive, got {bw}")
    t.link_bw = bw
    return Problem(dag, profiles, ids, rank, t)


def _pset(vals):
    vals = tuple(int(x) for x in vals)
    if not vals:
        raise ValueError("empty parallelism set")
    if len(vals) > abi.MAX_P:
        raise ValueError(f"more than {abi.MAX_P} parallelism options")
    if min(vals) < 1:
        raise ValueError("P, R and B must all be >= 1")
    return vals


def pack_grid(problem: Problem, params, bounds) -> abi.OpscGrid:
    """Menus of brute_force_autoscale: per op P asc, R in 1..r_max, B in 1..b_max."""
    g = abi.OpscGrid()
    if bounds.r_max < 1:
        raise ValueError("min() arg is an empty sequence")  # reference: empty menu
    g.r_max = int(bounds.r_max)
    off = 0
    for v, op in enumerate(problem.ids):
        pv = _pset(bounds.parallelism_for(params, op))
        bm = int(bounds.b_max_for(params, op))
        if bm < 1:
            raise ValueError("min() arg is an empty sequence")
        g.n_p[v] = len(pv)
        for i, p in enumerate(pv):
            g.p_vals[v][i] = p
        g.b_max[v] = bm
        g.menu_off[v] = off
        off += len(pv) * g.r_max * bm
        qv = _pset(params.parallelism_for(op))
        g.params_n_p[v] = len(qv)
        for i, p in enumerate(qv):
            g.params_p_vals[v][i] = p
        g.params_b_max[v] = int(params.b_max_for(op))
    g.menu_off[problem.n_ops] = off
    g.r_cap = int(params.r_cap)
    return g


def menu_sizes(problem: Problem, grid: abi.OpscGrid):
    return [grid.menu_off[v + 1] - grid.menu_off[v] for v in range(problem.n_ops)]


def pack_model(problem: Problem, params) -> abi.OpscModelSpec:
    """model_level_autoscale grid (autoscaler.py:612-615)."""
    s = abi.OpscModelSpec()
    for v, op in enumerate(problem.ids):
        s.p_base[v] = _pset(params.parallelism_for(op))[0]
    s.b_cap = int(min(params.b_max_for(op) for op in problem.ids))
    s.r_cap = int(params.r_cap)
    return s


def pack_greedy(problem: Problem, params) -> abi.OpscGreedySpec:
    """greedy_autoscale knobs (AutoscaleParams) + the model-level grid of its
    uniform reseed (autoscaler.py:357-367)."""
    s = abi.OpscGreedySpec()
    for v, op in enumerate(problem.ids):
        pv = _pset(params.parallelism_for(op))
        s.n_p[v] = len(pv)
        for i, p in enumerate(pv):
            s.p_vals[v][i] = p
        s.b_max[v] = int(params.b_max_for(op))
    s.r_cap = int(params.r_cap)
    s.max_iterations = int(getattr(params, "max_iterations", 10_000))
    s.prune_excess_replicas = int(bool(getattr(params, "prune_excess_replicas", False)))
    s.model = pack_model(problem, params)
    return s


@dataclass
class PlaceInputs:
    spec: abi.OpscPlaceSpec
    mem_cap: np.ndarray  # keeps the buffer alive


def pack_place(fleet=None, energy=None) -> PlaceInputs:
    """Default-stream placement fleet (devices in sorted-id order,
    placement.py:155-156) and Eq. 9 coefficients (metrics.py:34-47)."""
    if fleet is None:
        caps = np.array([180e9], dtype=np.float64)
        n_dev, uniform = 1 << 20, 1
    else:
        devs = sorted(fleet, key=lambda d: d.id)
        caps = np.array([float(d.mem_cap) for d in devs], dtype=np.float64)
        n_dev = len(devs)
        uniform = int(bool(n_dev) and bool(np.all(caps == caps[0])))
        if not n_dev:
            raise ValueError("fleet must not be empty")
    s = abi.OpscPlaceSpec()
    s.n_devices = n_dev
    s.uniform_cap = uniform
    s.alpha = float(energy.alpha) if energy is not None else 0.3 * 400.0
    s.beta = float(energy.beta) if energy is not None else 0.7 * 400.0
    s.mem_cap = caps.ctypes.data
    return PlaceInputs(s, caps)


@dataclass
class WindowArrays:
    qps: np.ndarray
    seq_len: np.ndarray
    phase: np.ndarray
    slo: np.ndarray
    eps: np.ndarray

    @property
    def n(self):
        return int(self.qps.shape[0])

    def struct(self) -> abi.OpscWindows:
        """The C-ABI view (cached while the same arrays are attached: building
        it costs ~10 us of numpy attribute lookups per call)."""
        arrs = (self.qps, self.seq_len, self.phase, self.slo, self.eps)
        hit = self.__dict__.get("_struct")
        if hit is not None and all(map(is_, hit[0], arrs)):
            return hit[1]
        w = abi.OpscWindows()
        w.n = self.n
        w.qps, w.seq_len, w.phase = self.qps.ctypes.data, self.seq_len.ctypes.data, self.phase.ctypes.data
        w.slo, w.eps = self.slo.ctypes.data, self.eps.ctypes.data
        self.__dict__["_struct"] = (arrs, w)
        return w

    def take(self, idx):
        return WindowArrays(*(np.ascontiguousarray(a[idx]) for a in
                              (self.qps, self.seq_len, self.phase, self.slo, self.eps)))


def pack_windows(points, slo, eps) -> WindowArrays:
    """WorkloadPoints (workload.py:38-54) + per-window SLO/epsilon as SoA."""
    n = len(points)
    slo = np.broadcast_to(np.asarray(slo, dtype=np.float64), (n,))
    eps = np.broadcast_to(np.asarray(eps, dtype=np.float64), (n,))
    return WindowArrays(
        qps=np.array([float(p.qps) for p in points], dtype=np.float64),
        seq_len=np.array([int(p.seq_len) for p in points], dtype=np.int32),
        phase=np.array([PHASE_INDEX[p.phase] for p in points], dtype=np.uint8),
        slo=np.ascontiguousarray(slo), eps=np.ascontiguousarray(eps),
    )


def window_arrays(qps, seq_len, phase, slo, eps=0.0) -> WindowArrays:
    n = len(qps)
    ph = np.broadcast_to(np.asarray(phase, dtype=np.uint8), (n,))
    return WindowArrays(
        qps=np.ascontiguousarray(qps, dtype=np.float64),
        seq_len=np.ascontiguousarray(seq_len, dtype=np.int32),
        phase=np.ascontiguousarray(ph),
        slo=np.ascontiguousarray(np.broadcast_to(np.asarray(slo, np.float64), (n,))),
        eps=np.ascontiguousarray(np.broadcast_to(np.asarray(eps, np.float64), (n,))),
    )


TRACE_DTYPE = np.dtype([("latency", "<f8"), ("objective", "<i4"), ("to_r", "<i2"),
                        ("to_b", "<i2"), ("to_p", "<i2"), ("op", "i1"), ("action", "u1"),
                        ("reserved", "<i4")], align=True)
assert TRACE_DTYPE.itemsize == C.sizeof(abi.OpscTraceEntry)


class DecisionArrays:
    """Host SoA of OpscDecisions for W windows x n ops."""

    def __init__(self, n_windows, n_ops, trace_cap=0):
        W, n = n_windows, n_ops
        self.n_windows, self.n_ops = W, n
        self.key = np.full(W, abi.KEY_INFEASIBLE, dtype=np.int64)
        self.cfg = np.zeros((W, n, 3), dtype=np.int16)
        self.feasible = np.zeros(W, dtype=np.uint8)
        self.status = np.zeros(W, dtype=np.uint32)
        self.latency = np.zeros(W, dtype=np.float64)
        self.objective = np.zeros(W, dtype=np.int32)
        self.path = np.full((W, n), -1, dtype=np.int8)
        self.pred = np.zeros((W, n, abi.PRED_FIELDS), dtype=np.float64)
        self.stable = np.zeros((W, n), dtype=np.uint8)
        self.energy = np.zeros(W, dtype=np.float64)
        self.memory = np.zeros(W, dtype=np.float64)
        self.devices = np.zeros(W, dtype=np.int32)
        self.trace_cap = int(trace_cap)
        self.trace_len = np.zeros(W, dtype=np.int32)
        self.trace = np.zeros((W, max(self.trace_cap, 1)), dtype=TRACE_DTYPE)

    FIELDS = ("key", "cfg", "feasible", "status", "latency", "objective", "path",
              "pred", "stable", "energy", "memory", "devices")

    def struct(self) -> abi.OpscDecisions:
        """The C-ABI view (cached while the same arrays are attached)."""
        arrs = tuple(getattr(self, f) for f in self.FIELDS) + (self.trace_len, self.trace)
        hit = self.__dict__.get("_struct")
        if hit is not None and hit[2] == self.trace_cap and all(map(is_, hit[0], arrs)):
            return hit[1]
        d = abi.OpscDecisions()
        for f in self.FIELDS:
            setattr(d, f, getattr(self, f).ctypes.data)
        d.trace_cap = self.trace_cap
        d.trace_len = self.trace_len.ctypes.data
        d.trace = self.trace.ctypes.data
        self.__dict__["_struct"] = (arrs, d, self.trace_cap)
        return d

    def nbytes(self):
        n = sum(getattr(self, f).nbytes for f in self.FIELDS)
        return n + (self.trace_len.nbytes + self.trace.nbytes if self.trace_cap else 0)

    def with_trace_cap(self, cap):
        """A copy whose move-trace rows hold `cap` entries (existing entries kept)."""
        out = DecisionArrays(self.n_windows, self.n_ops, cap)
        for f in self.FIELDS + ("trace_len",):
            getattr(out, f)[...] = getattr(self, f)
        k = min(self.trace_cap, cap)
        out.trace[:, :k] = self.trace[:, :k]
        return out

    def splice(self, idx, other):
        """Rows `idx` replaced by `other`'s rows 0..len(idx)-1 (trace_cap of
        self must hold other's entries)."""
        for f in self.FIELDS + ("trace_len",):
            getattr(self, f)[idx] = getattr(other, f)
        if self.trace_cap:
            k = min(self.trace_cap, other.trace_cap)
            self.trace[idx, :k] = other.trace[:, :k]


def c_ptr(x):
    return C.byref(x)
