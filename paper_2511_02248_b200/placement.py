"""Shared (interference-aware) placement of decided plans -- Alg. 2 of the
reference (placement.py:399-462) -- and its Eq. 9 energy / memory metrics
(metrics.py:84-132), as packed C-ABI inputs and SoA outputs.

`place_windows` runs opsc_place_shared on the GPU (one CTA per window);
`placement_objects` turns the arrays into reference-shaped Placement objects.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import abi


class SharedFleet:
    """Fleet (devices sorted by id, placement.py:155-156) + PlacementParams +
    InterferenceParams + EnergyParams packed as an OpscPlaceShared."""

    def __init__(self, fleet, slo, interference=None, energy=None, slack_weight_mem=0.5,
                 slack_weight_compute=0.5, max_sm_load=1.5, default_stream=False, window_slo=False):
        if not fleet:
            raise ValueError("fleet must not be empty")
        self.devices = sorted(fleet, key=lambda d: d.id)
        self.mem_cap = np.array([float(d.mem_cap) for d in self.devices])
        self.compute_cap = np.array([float(getattr(d, "compute_cap", 1.0)) for d in self.devices])
        s = abi.OpscPlaceShared()
        s.n_devices = len(self.devices)
        s.mem_cap, s.compute_cap = self.mem_cap.ctypes.data, self.compute_cap.ctypes.data
        s.slo = float(slo)
        s.slack_weight_mem, s.slack_weight_compute = float(slack_weight_mem), float(slack_weight_compute)
        s.max_sm_load = float(max_sm_load)
        s.theta = float(interference.theta) if interference is not None else 0.5
        s.exponent = float(interference.exponent) if interference is not None else 1.0
        s.alpha = float(energy.alpha) if energy is not None else 0.3 * 400.0
        s.beta = float(energy.beta) if energy is not None else 0.7 * 400.0
        s.flags = (abi.PLACE_DEFAULT_STREAM if default_stream else 0) | (abi.PLACE_WINDOW_SLO if window_slo else 0)
        self.spec = s

    @classmethod
    def from_params(cls, fleet, placement_params, profiles, energy=None, **flags):
        p = placement_params
        return cls(fleet, p.slo, getattr(profiles, "interference", None), energy,
                   p.slack_weight_mem, p.slack_weight_compute, p.max_sm_load, **flags)


class PlacementArrays:
    """Host SoA of OpscPlacement for W windows."""

    FIELDS = ("n_assign", "devices_used", "feasible", "status", "latency", "energy", "memory",
              "a_op", "a_replica", "a_device", "a_share", "a_latency", "d_mem", "d_sm", "d_energy")

    def __init__(self, n_windows, cap_assign, cap_dev):
        W, A, D = n_windows, max(1, cap_assign), max(1, cap_dev)
        self.cap_assign, self.cap_dev = A, D
        self.n_assign = np.zeros(W, np.int32)
        self.devices_used = np.zeros(W, np.int32)
        self.feasible = np.zeros(W, np.uint8)
        self.status = np.zeros(W, np.uint32)
        self.latency = np.zeros(W)
        self.energy = np.zeros(W)
        self.memory = np.zeros(W)
        self.a_op = np.zeros((W, A), np.int8)
        self.a_replica = np.zeros((W, A), np.int16)
        self.a_device = np.zeros((W, A), np.int32)
        self.a_share = np.zeros((W, A), np.int16)
        self.a_latency = np.zeros((W, A))
        self.d_mem = np.zeros((W, D))
        self.d_sm = np.zeros((W, D))
        self.d_energy = np.zeros((W, D))

    def struct(self):
        s = abi.OpscPlacement()
        s.cap_assign, s.cap_dev = self.cap_assign, self.cap_dev
        for f in self.FIELDS:
            setattr(s, f, getattr(self, f).ctypes.data)
        return s


def capacities(cfg, n_devices):
    """Assignment / device slots needed by the plans in cfg [W][n][3]:
    every replica is one assignment and needs at most one device."""
    total_r = int(cfg[:, :, 1].sum(axis=1).max()) if cfg.size else 1
    return max(1, total_r), max(1, min(int(n_devices), total_r))


def place_windows(problem, windows, cfg, plan_feasible, fleet: SharedFleet, config_order,
                  device="cuda"):
    """opsc_place_shared on the GPU for every window's decided plan; host
    arrays in, PlacementArrays out."""
    import torch

    from . import _native, tables
    dev = torch.device(device)
    L = _native.load()
    cfg = np.ascontiguousarray(cfg, dtype=np.int16)
    ca, cd = capacities(cfg, fleet.spec.n_devices)
    host = PlacementArrays(windows.n, ca, cd)
    to = lambda a: torch.from_numpy(np.array(a, copy=True)).to(dev)
    wt = {k: to(getattr(windows, k)) for k in ("qps", "seq_len", "phase", "slo", "eps")}
    w = abi.OpscWindows()
    w.n = windows.n
    for k, t in wt.items():
        setattr(w, k, t.data_ptr())
    cfg_t, feas_t = to(cfg), to(np.ascontiguousarray(plan_feasible, dtype=np.uint8))
    caps_t, ccap_t = to(fleet.mem_cap), to(fleet.compute_cap)
    spec = abi.OpscPlaceShared()
    for f, _ in abi.OpscPlaceShared._fields_:
        setattr(spec, f, getattr(fleet.spec, f))
    spec.mem_cap, spec.compute_cap = caps_t.data_ptr(), ccap_t.data_ptr()
    dt = {f: to(getattr(host, f)) for f in PlacementArrays.FIELDS}
    out = abi.OpscPlacement()
    out.cap_assign, out.cap_dev = host.cap_assign, host.cap_dev
    for f, t in dt.items():
        setattr(out, f, t.data_ptr())
    nb = L.opsc_place_shared_workspace(windows.n, host.cap_assign, host.cap_dev, problem.n_ops)
    ws = torch.empty(nb, dtype=torch.uint8, device=dev)
    _native.check(L.opsc_place_shared(_native.ref(problem.table), _native.ref(spec), w, cfg_t.data_ptr(),
                                      feas_t.data_ptr(), config_order, out, ws.data_ptr(), nb,
                                      torch.cuda.current_stream(dev).cuda_stream), "opsc_place_shared")
    torch.cuda.synchronize(dev)
    for f, t in dt.items():
        getattr(host, f)[...] = t.cpu().numpy()
    return host


def placement_object(arr, i, plan, dag, profiles, problem, fleet: SharedFleet, seq_len, types):
    """Window i of PlacementArrays as the reference's Placement
    (placement.py:59-110): assignments in placement order with
    interference-adjusted latency, device loads (sorted-id order) carrying
    fill_device_energy's per-device energy."""
    T = types
    L = int(seq_len)
    k_base = min(c.r for c in plan.configs.values())
    assignments = []
    for a in range(int(arr.n_assign[i])):
        op = problem.ids[int(arr.a_op[i, a])]
        c = plan.configs[op]
        prof = profiles.get(dag.node(op).profile_ref)
        k = int(arr.a_replica[i, a])
        assignments.append(T.ReplicaAssignment(
            op_id=op, replica_index=k, device_id=fleet.devices[int(arr.a_device[i, a])].id,
            sm_share=int(arr.a_share[i, a]), sm_demand=min(1.0, prof.s0 + prof.s1 * c.b * L),
            mem_bytes=prof.weight_mem / c.p + prof.m0 + prof.m1 * c.b * L,
            group=f"base{k}" if k <= k_base else f"extra:{op}:{k}",
            interference_adjusted_latency=float(arr.a_latency[i, a])))
    loads = {fleet.devices[d].id: T.DeviceLoad(mem_used=float(arr.d_mem[i, d]),
                                               sm_demand=float(arr.d_sm[i, d]),
                                               energy=float(arr.d_energy[i, d]))
             for d in range(int(arr.devices_used[i]))}
    return T.Placement(assignments=assignments, device_loads=loads,
                       devices_used=int(arr.devices_used[i]), feasible=bool(arr.feasible[i]),
                       recomputed_latency=float(arr.latency[i]))


def raise_placement_status(status, n_devices, err):
    if status & abi.W_FLEET_EXHAUSTED:
        raise err.FleetExhausted(f"all {n_devices} devices in use, none left to provision")
    if status & abi.W_INFEASIBLE_PLACEMENT:
        raise err.InfeasiblePlacement("a replica needs more memory than its device holds")


def _place_one(plan, dag, profiles, fleet, params, point, types, err, energy, return_metrics,
               default_stream):
    from . import errors, model, tables
    T = types or model
    E = err or errors
    if not plan.feasible:
        raise ValueError("placement requires an SLO-feasible plan")
    if not fleet:
        raise ValueError("fleet must not be empty")
    problem = tables.pack_problem(dag, profiles)
    # the plan's config order drives the energy sum (metrics.py:95-101)
    order = [problem.rank[op] for op in plan.configs]
    C.memmove(C.addressof(problem.table) + abi.OpscDag.node_order.offset,
              (C.c_int32 * len(order))(*order), 4 * len(order))
    cfg = np.zeros((1, problem.n_ops, 3), np.int16)
    for op, c in plan.configs.items():
        cfg[0, problem.rank[op]] = (c.p, c.r, c.b)
    win = tables.pack_windows([point], params.slo, 0.0)
    sf = SharedFleet.from_params(fleet, params, profiles, energy, default_stream=default_stream)
    arr = place_windows(problem, win, cfg, np.ones(1, np.uint8), sf, 1)
    raise_placement_status(int(arr.status[0]), len(fleet), E)
    placed = placement_object(arr, 0, plan, dag, profiles, problem, sf, point.seq_len, T)
    if return_metrics:
        return placed, float(arr.energy[0]), float(arr.memory[0])
    return placed


def place(plan, dag, profiles, fleet, params, point, *, types=None, err=None, energy=None,
          return_metrics=False):
    """Drop-in for the reference's placement.place() (placement.py:399-462):
    Alg. 2 on the GPU for one decided plan. Returns a Placement whose
    device_loads already carry fill_device_energy's per-device energy; with
    return_metrics=True also (request_energy, provisioned_memory)."""
    return _place_one(plan, dag, profiles, fleet, params, point, types, err, energy, return_metrics, False)


def default_stream_place(plan, dag, profiles, fleet, params, point, *, types=None, err=None,
                         energy=None, return_metrics=False):
    """Drop-in for default_stream_place() (placement.py:465-491): the same
    base instances, every extra replica on a dedicated device."""
    return _place_one(plan, dag, profiles, fleet, params, point, types, err, energy, return_metrics, True)
