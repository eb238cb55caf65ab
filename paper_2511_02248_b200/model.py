"""Host-side planning data model, mirroring the reference API surface.

These are the value types the planners consume and produce. They keep the
reference's names, fields and validation errors so code written against the
reference (`opscaler`) reads the same here:

  OperatorNode / Edge / OperatorDag / build_dag   opgraph.py:41-171
  LatencyModel / OperatorProfile / ProfileSet     perfmodel.py:49-130
  profiles_from_dict                              perfmodel.py:311-324
  WorkloadPoint                                   workload.py:38-54
  OperatorConfig / PredictedSojourn / ScalingPlan autoscaler.py:44-99
  AutoscaleParams / BruteForceBounds              autoscaler.py:102-131, 688-700
  EnergyParams                                    metrics.py:34-47
  DeviceSpec / make_fleet                         placement.py:46-55, 135-140

None of this is on the device path: the planners only read these objects
(duck-typed, so the reference's own instances work too) and pack them into
the C-ABI tables of `tables.py`.
"""

from __future__ import annotations

import heapq
from dataclasses import dataclass, field

from .errors import CycleDetected, DanglingEdge, UnknownPhase, UnknownProfile

PHASES = ("prefill", "decode")
OPERATOR_KINDS = (
    "attention", "linear", "moe_linear", "norm", "activation",
    "embedding", "elementwise", "other",
)
DEFAULT_PARALLELISM = (1, 2, 4, 8)


# --------------------------------------------------------------------------
# graph


@dataclass(frozen=True)
class OperatorNode:
    id: str
    kind: str
    layer_count: int = 1
    profile_ref: str = ""

    def __post_init__(self):
        if self.layer_count < 1:
            raise ValueError(f"node {self.id}: layer_count must be >= 1")
        if self.kind not in OPERATOR_KINDS:
            raise ValueError(f"node {self.id}: unknown kind {self.kind!r}")


@dataclass(frozen=True)
class Edge:
    src: str
    dst: str
    volume_ref: str = ""


@dataclass
class OperatorDag:
    """Validated operator graph; topological order is Kahn's algorithm with
    the ready set kept sorted by id (the reference's order, opgraph.py:110-132)."""

    nodes: list
    edges: list
    sources: list = field(default_factory=list)
    sinks: list = field(default_factory=list)
    topo_order: list = field(default_factory=list)

    def __post_init__(self):
        self._by_id = {}
        for n in self.nodes:
            if n.id in self._by_id:
                raise ValueError(f"duplicate node id {n.id!r}")
            self._by_id[n.id] = n
        succ = {n.id: [] for n in self.nodes}
        pred = {n.id: [] for n in self.nodes}
        for e in self.edges:
            for end in (e.src, e.dst):
                if end not in self._by_id:
                    raise DanglingEdge(
                        f"edge ({e.src} -> {e.dst}) references missing node {end!r}")
            succ[e.src].append(e.dst)
            pred[e.dst].append(e.src)
        self._succ = {k: sorted(v) for k, v in succ.items()}
        self._pred = {k: sorted(v) for k, v in pred.items()}
        self.topo_order = self._kahn()
        self.sources = sorted(k for k, v in self._pred.items() if not v)
        self.sinks = sorted(k for k, v in self._succ.items() if not v)
        if not self.sources or not self.sinks:
            raise CycleDetected("graph has no source or no sink")

    def _kahn(self):
        indeg = {k: len(v) for k, v in self._pred.items()}
        heap = [k for k, d in indeg.items() if d == 0]
        heapq.heapify(heap)
        order = []
        while heap:
            v = heapq.heappop(heap)
            order.append(v)
            for w in self._succ[v]:
                indeg[w] -= 1
                if indeg[w] == 0:
                    heapq.heappush(heap, w)
        if len(order) != len(self.nodes):
            stuck = sorted(k for k, d in indeg.items() if d > 0)
            raise CycleDetected(f"cycle through nodes {stuck}")
        return order

    def node(self, node_id):
        return self._by_id[node_id]

    def successors(self, node_id):
        return self._succ[node_id]

    def predecessors(self, node_id):
        return self._pred[node_id]

    def out_edges(self, node_id):
        return [e for e in self.edges if e.src == node_id]

    @property
    def node_ids(self):
        return [n.id for n in self.nodes]


def build_dag(spec: dict) -> OperatorDag:
    """{"nodes": [{"id", "kind", "layer_count", "profile_ref"}], "edges":
    [{"src", "dst", "volume_ref"}]} -> OperatorDag (opgraph.py:151-171)."""
    nodes = [
        OperatorNode(
            id=n["id"], kind=n.get("kind", "other"),
            layer_count=int(n.get("layer_count", 1)),
            profile_ref=n.get("profile_ref", n["id"]),
        )
        for n in spec.get("nodes", [])
    ]
    edges = [
        Edge(src=e["src"], dst=e["dst"], volume_ref=e.get("volume_ref", e["src"]))
        for e in spec.get("edges", [])
    ]
    return OperatorDag(nodes=nodes, edges=edges)


# --------------------------------------------------------------------------
# profiles


@dataclass(frozen=True)
class LatencyModel:
    c0: float = 0.0
    c1: float = 0.0
    c2: float = 0.0

    def __post_init__(self):
        if self.c0 < 0 or self.c1 < 0 or self.c2 < 0:
            raise ValueError("latency coefficients must be non-negative")


@dataclass(frozen=True)
class InterferenceParams:
    theta: float = 0.5
    exponent: float = 1.0


@dataclass(frozen=True)
class OperatorProfile:
    name: str
    phase_models: dict
    weight_mem: float = 0.0
    m0: float = 0.0
    m1: float = 0.0
    v0: float = 0.0
    v1: float = 0.0
    s0: float = 0.0
    s1: float = 0.0
    eta: float = 0.9
    kind: str = "other"

    def __post_init__(self):
        for name in ("weight_mem", "m0", "m1", "v0", "v1", "s0", "s1"):
            if getattr(self, name) < 0:
                raise ValueError(f"{self.name}: {name} must be >= 0")
        if not (0.0 < self.eta <= 1.0):
            raise ValueError(f"{self.name}: eta must be in (0, 1]")

    def latency_model(self, phase):
        if phase not in PHASES:
            raise UnknownPhase(f"unknown phase {phase!r}")
        if phase not in self.phase_models:
            raise UnknownPhase(f"profile {self.name} has no {phase} model")
        return self.phase_models[phase]


@dataclass
class ProfileSet:
    profiles: dict
    link_bandwidth: float = 600e9
    interference: InterferenceParams = field(default_factory=InterferenceParams)

    def get(self, name):
        try:
            return self.profiles[name]
        except KeyError:
            raise UnknownProfile(f"no profile named {name!r}") from None

    def validate_against(self, dag):
        for n in dag.nodes:
            self.get(n.profile_ref)
        for e in dag.edges:
            self.get(e.volume_ref)


def profiles_from_dict(raw: dict) -> ProfileSet:
    """Profile JSON schema of the reference (perfmodel.py:300-324): name ->
    {phase: {c0, c1, c2}, weight_mem, m0, m1, v0, v1, s0, s1, eta, kind};
    keys starting with "_" are set-level (_link_bandwidth, _interference)."""
    inter = raw.get("_interference", {})
    profiles = {}
    for name, body in raw.items():
        if name.startswith("_"):
            continue
        models = {
            ph: LatencyModel(float(body[ph].get("c0", 0.0)),
                             float(body[ph].get("c1", 0.0)),
                             float(body[ph].get("c2", 0.0)))
            for ph in PHASES if ph in body
        }
        profiles[name] = OperatorProfile(
            name=name, phase_models=models,
            **{k: float(body.get(k, 0.0))
               for k in ("weight_mem", "m0", "m1", "v0", "v1", "s0", "s1")},
            eta=float(body.get("eta", 0.9)), kind=body.get("kind", "other"),
        )
    return ProfileSet(
        profiles=profiles,
        link_bandwidth=float(raw.get("_link_bandwidth", 600e9)),
        interference=InterferenceParams(float(inter.get("theta", 0.5)),
                                        float(inter.get("exponent", 1.0))),
    )


# --------------------------------------------------------------------------
# workload


@dataclass(frozen=True)
class WorkloadPoint:
    qps: float
    seq_len: int
    phase: str
    window: tuple = (0.0, 0.0)

    def __post_init__(self):
        if self.qps < 0:
            raise ValueError("qps must be >= 0")
        if self.seq_len < 1:
            raise ValueError("seq_len must be >= 1")
        if self.phase not in PHASES:
            raise ValueError(f"unknown phase {self.phase!r}")


# --------------------------------------------------------------------------
# plans and planner knobs


@dataclass(frozen=True)
class OperatorConfig:
    p: int
    r: int
    b: int
    sm_share: int = 100

    def __post_init__(self):
        if self.p < 1 or self.r < 1 or self.b < 1:
            raise ValueError("P, R and B must all be >= 1")
        if not (1 <= self.sm_share <= 100):
            raise ValueError(f"sm_share must be in [1, 100], got {self.sm_share}")


@dataclass(frozen=True)
class PredictedSojourn:
    op_latency: float
    lam: float
    mu: float
    utilization: float
    wait: float
    service: float
    comm: float
    stable: bool

    @property
    def sojourn(self) -> float:
        return self.wait + self.service


@dataclass
class ScalingPlan:
    configs: dict
    predicted: dict
    iteration_latency: float
    critical_path: list
    objective: int
    feasible: bool
    phase: str
    trace: list = field(default_factory=list)

    def to_dict(self) -> dict:
        return {
            "operators": {op: {"P": c.p, "R": c.r, "B": c.b, "sm_share": c.sm_share}
                          for op, c in sorted(self.configs.items())},
            "iteration_latency": self.iteration_latency,
            "critical_path": self.critical_path,
            "objective": self.objective,
            "feasible": self.feasible,
            "phase": self.phase,
            "trace": self.trace,
        }


@dataclass(frozen=True)
class AutoscaleParams:
    slo: float
    epsilon: float = 0.0
    b_max: object = 32
    parallelism: object = DEFAULT_PARALLELISM
    r_cap: int = 512
    max_iterations: int = 10_000
    prune_excess_replicas: bool = False

    def __post_init__(self):
        if self.slo <= 0:
            raise ValueError("slo must be positive")
        if not (0 <= self.epsilon < self.slo):
            raise ValueError("epsilon must satisfy 0 <= epsilon < slo")

    def b_max_for(self, op_id):
        return self.b_max[op_id] if isinstance(self.b_max, dict) else self.b_max

    def parallelism_for(self, op_id):
        opts = (self.parallelism[op_id] if isinstance(self.parallelism, dict)
                else self.parallelism)
        return tuple(sorted(opts))


@dataclass(frozen=True)
class BruteForceBounds:
    r_max: int = 8
    b_max: int | None = None
    parallelism: tuple | None = None

    def b_max_for(self, params, op_id):
        return self.b_max if self.b_max is not None else params.b_max_for(op_id)

    def parallelism_for(self, params, op_id):
        if self.parallelism is not None:
            return tuple(sorted(self.parallelism))
        return params.parallelism_for(op_id)


REFERENCE_GPU_WATTS = 400.0


@dataclass(frozen=True)
class EnergyParams:
    alpha: float = 0.3 * REFERENCE_GPU_WATTS
    beta: float = 0.7 * REFERENCE_GPU_WATTS

    def __post_init__(self):
        if self.alpha < 0 or self.beta < 0:
            raise ValueError("power coefficients must be >= 0")


@dataclass(frozen=True)
class DeviceSpec:
    id: str
    mem_cap: float = 80e9
    compute_cap: float = 1.0
    link_bw: float = 600e9

    def __post_init__(self):
        if self.mem_cap <= 0:
            raise ValueError(f"device {self.id}: mem_cap must be positive")


def make_fleet(n: int, mem_cap: float = 80e9, link_bw: float = 600e9):
    width = len(str(max(0, n - 1)))
    return [DeviceSpec(id=f"gpu{i:0{width}d}", mem_cap=mem_cap, link_bw=link_bw)
            for i in range(n)]


# --------------------------------------------------------------------------
# placement value types (placement.py:58-117)


@dataclass
class ReplicaAssignment:
    op_id: str
    replica_index: int
    device_id: str
    sm_share: int
    sm_demand: float
    mem_bytes: float
    group: str
    interference_adjusted_latency: float = 0.0


@dataclass
class DeviceLoad:
    mem_used: float = 0.0
    sm_demand: float = 0.0
    energy: float = 0.0


@dataclass
class Placement:
    assignments: list
    device_loads: dict
    devices_used: int
    feasible: bool
    recomputed_latency: float

    def to_dict(self) -> dict:
        """Same keys and order as the reference's Placement.to_dict
        (placement.py:85-110); devices sorted by id."""
        return {
            "assignments": [{"op": a.op_id, "replica": a.replica_index, "device": a.device_id,
                             "sm_share": a.sm_share,
                             "interference_adjusted_latency": a.interference_adjusted_latency}
                            for a in self.assignments],
            "devices": [{"id": dev, "mem_used": ld.mem_used, "sm_demand": ld.sm_demand,
                         "energy": ld.energy}
                        for dev, ld in sorted(self.device_loads.items())],
            "devices_used": self.devices_used,
            "feasible": self.feasible,
            "recomputed_latency": self.recomputed_latency,
        }


@dataclass(frozen=True)
class PlacementParams:
    slo: float
    slack_weight_mem: float = 0.5
    slack_weight_compute: float = 0.5
    max_sm_load: float = 1.5
