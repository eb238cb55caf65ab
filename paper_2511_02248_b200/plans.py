"""Turn per-window decision arrays into reference-shaped ScalingPlans.

The device path returns structure-of-arrays decisions (OpscDecisions); this
module maps them back onto the planner API: OperatorConfig / PredictedSojourn
/ ScalingPlan objects (autoscaler.py:44-99, _make_plan :231-247) and the
reference's exceptions, raised in the order the reference would hit them
(autoscaler.py:706-847 for the oracle, :596-681 for the model level).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

from . import abi, errors, model

# config dict order per mode: brute force builds configs in sorted-id order
# (autoscaler.py:825, 843-845); the model level in dag.node_ids order (:617-618)
ORDER_LEX, ORDER_NODE = 0, 1


def _op_named(status, shift, problem, node_order):
    """The operator id the device recorded in a status word's op field."""
    k = (status >> shift) & abi.W_OP_FIELD
    if not k or problem is None:
        return "?"
    rank = problem.table.node_order[k - 1] if node_order else k - 1
    return problem.ids[rank]


def raise_for_status(status: int, mode: int, err=errors, *, problem=None, qps=None, r_cap=None):
    """Raise the reference's exception (class and text) for a window status.

    The texts are the reference's: init_configs (autoscaler.py:289-292, also
    reached by brute force through its greedy warm start, :771), the
    brute-force bounds fallback (:835-837), model level (:678-681) and
    erlang_c on a utilization that rounds to 1 (queueing.py:68-69)."""
    if status & abi.W_ZERO_DIVISION:
        raise ZeroDivisionError("float division by zero")
    if status & abi.W_UNSTABLE_ROUNDING:
        raise err.Unstable("utilization 1.0 >= 1: queue has no steady state")
    init_msg = lambda: (f"operator {_op_named(status, abi.W_INIT_OP_SHIFT, problem, True)}: "
                        f"arrival rate {qps} exceeds capacity at every (B, P) within r_cap={r_cap}")
    if mode == abi.MODE_ORACLE:
        if status & abi.W_NO_STABLE_PARAMS:
            raise err.NoStableConfig(init_msg())
        if status & abi.W_NO_STABLE_BOUNDS:
            op = _op_named(status, abi.W_BOUNDS_OP_SHIFT, problem, False)
            raise err.NoStableConfig(f"operator {op}: no stable configuration within bounds")
    elif mode == abi.MODE_OPERATOR:
        if status & abi.W_NO_STABLE_INIT:
            raise err.NoStableConfig(init_msg())
        if status & abi.W_TRACE_TRUNCATED:
            raise RuntimeError("greedy move trace exceeded trace_cap; raise trace_cap")
    elif status & abi.W_NO_STABLE_MODEL:
        raise err.NoStableConfig(
            f"model-level: arrival rate {qps} exceeds capacity at every batch size within r_cap={r_cap}")


def nonfinite_qps(qps):
    """A NaN / +inf arrival rate passes the reference's `qps <= 0` check
    (autoscaler.py:148) and fails in _strict_min_replicas' math.ceil
    (autoscaler.py:225), reached by every planner; the device treats such a
    window as idle, so the host raises the reference's error here."""
    if math.isnan(qps):
        raise ValueError("cannot convert float NaN to integer")
    if math.isinf(qps) and qps > 0:
        raise OverflowError("cannot convert float infinity to integer")


def _builder(cls, names):
    """Fast constructor for the plan's value types (OperatorConfig,
    PredictedSojourn, ScalingPlan -- this package's or the reference's,
    autoscaler.py:44-99): fills the instance dict directly, skipping
    dataclass __init__ / __post_init__, whose checks (P, R, B >= 1) the device
    results satisfy by construction. Equality, hash and repr are the
    dataclass's own. The body is generated for the class's field names (one
    dict store per field: ~3x faster than dict.update(zip(...))). Classes
    without an instance dict fall back to the normal constructor."""
    probe = object.__new__(cls)
    if not hasattr(probe, "__dict__") or not all(n.isidentifier() for n in names):
        return cls
    args = ", ".join(f"v{i}" for i in range(len(names)))
    body = "".join(f"    d[{n!r}] = v{i}\n" for i, n in enumerate(names))
    src = f"def make({args}):\n    o = new(cls)\n    d = o.__dict__\n{body}    return o\n"
    ns = {"new": object.__new__, "cls": cls}
    exec(src, ns)  # noqa: S102 -- field names are the dataclass's own identifiers
    return ns["make"]


_BUILDERS = {}


def builders(T):
    """(OperatorConfig factory, PredictedSojourn factory, ScalingPlan factory)
    of a type namespace. OperatorConfig is a frozen value type with a small
    domain, so its factory hands out one shared instance per (P, R, B)
    (as immutable as the ones the reference creates per plan)."""
    b = _BUILDERS.get(id(T))
    if b is None or b[0] is not T:
        import dataclasses
        oc = T.OperatorConfig
        ps = T.PredictedSojourn
        sp = T.ScalingPlan
        mk_oc = _builder(oc, [f.name for f in dataclasses.fields(oc)])
        frozen = getattr(getattr(oc, "__dataclass_params__", None), "frozen", False)
        if frozen:
            cache = {}

            def make_oc(p, r, b_, share, _c=cache, _mk=mk_oc):
                k = (p << 42) | (r << 21) | b_
                o = _c.get(k)
                if o is None:
                    o = _c[k] = _mk(p, r, b_, share)
                return o
        else:
            make_oc = mk_oc
        b = (T, make_oc, _builder(ps, [f.name for f in dataclasses.fields(ps)]),
             _builder(sp, [f.name for f in dataclasses.fields(sp)]))
        _BUILDERS[id(T)] = b
    return b[1], b[2], b[3]


@dataclass
class PlanMetrics:
    """Default-stream placement figures of a feasible plan (runner.py:94-96)."""

    devices_used: int
    energy_joules: float
    memory_bytes: float
    error: str | None = None


class WindowDecisions:
    """Decisions for a batch of windows, with lazy plan materialisation."""

    def __init__(self, problem, points, arrays, mode, types=model, err=errors, r_cap=None):
        self.problem, self.points, self.arrays, self.mode = problem, points, arrays, mode
        self.types, self.err = types, err
        self.r_cap = r_cap  # AutoscaleParams.r_cap, for the NoStableConfig texts

    def __len__(self):
        return self.arrays.n_windows

    def status(self, i):
        return int(self.arrays.status[i])

    def order_sensitive(self, i):
        """True if the opt-in certificate (decide_windows(certify=True)) found
        that window i's brute-force decision could depend on the reference's
        leaf summation order (OPSC_W_ORDER_SENSITIVE)."""
        return bool(self.arrays.status[i] & abi.W_ORDER_SENSITIVE)

    def plan(self, i):
        a, ids = self.arrays, self.problem.ids
        st = int(a.status[i])
        qps = self.points[i].qps
        nonfinite_qps(qps)
        if st & abi.W_IDLE:
            return None
        if st:
            raise_for_status(st, self.mode, self.err, problem=self.problem, qps=qps, r_cap=self.r_cap)
        order = range(self.problem.n_ops) if self.mode == abi.MODE_ORACLE else self.problem.node_order
        cfg, pred, stable = a.cfg[i].tolist(), a.pred[i].tolist(), a.stable[i].tolist()
        OC, PS, SP = builders(self.types)
        configs, predicted = {}, {}
        for v in order:
            p, r, b = cfg[v]
            op = ids[v]
            configs[op] = OC(p, r, b, 100)  # sm_share: planners run at 100 (autoscaler.py:50)
            predicted[op] = PS(*pred[v], stable[v] != 0)
        lat = float(a.latency[i])
        path = [ids[x] for x in a.path[i].tolist() if x >= 0] if math.isfinite(lat) else []
        return SP(configs, predicted, lat, path, int(a.objective[i]), bool(a.feasible[i]),
                  self.points[i].phase, self.trace(i))

    def trace(self, i):
        """ScalingPlan.trace of the greedy planner (autoscaler.py:363, 446-454,
        478-486, 549-557, 579-587); empty for the other planners."""
        a = self.arrays
        if self.mode != abi.MODE_OPERATOR or not a.trace_cap:
            return []
        out = []
        ids = self.problem.ids
        for lat, obj, r, b, p, op, act, _ in a.trace[i, :min(int(a.trace_len[i]), a.trace_cap)].tolist():
            name = abi.ACTION_NAMES[act]
            if name == "reseed_uniform":
                out.append({"action": name, "objective": obj})
            else:
                out.append({"action": name, "op": ids[op], "to": {"R": r, "B": b, "P": p},
                            "latency": lat, "objective": obj})
        return out

    def plans(self):
        return [self.plan(i) for i in range(len(self))]

    def metrics(self, i):
        a = self.arrays
        st = int(a.status[i])
        if not a.feasible[i] or st & abi.W_IDLE:
            return None
        error = None
        if st & abi.W_FLEET_EXHAUSTED:
            error = "FleetExhausted"
        elif st & abi.W_INFEASIBLE_PLACEMENT:
            error = "InfeasiblePlacement"
        return PlanMetrics(int(a.devices[i]), float(a.energy[i]), float(a.memory[i]), error)
