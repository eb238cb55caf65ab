"""GPU shared placement (csrc/k_place.cu) against the reference's own
place()/energy outputs (golden) and the CPU oracle on large plans."""

import numpy as np
import pytest

import golden_cases as G
import test_oracle_place as TP
from paper_2511_02248_b200 import abi, model, placement, tables
from workloads import scenarios

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("variant", ["settings", "default_stream"])
def test_gpu_place_golden(variant):
    errs = []
    for rec in TP.CASES:
        e = TP.check_place(placement.place_windows, rec, TP.SETTINGS, variant)
        if e:
            errs.append((rec["name"], e[:2]))
    assert not errs, errs[:3]


def test_gpu_place_vs_oracle_large_plans(orc):
    """Model-level and greedy plans of the 70B trace (tens of replicas per op)."""
    from paper_2511_02248_b200 import _native
    prob = tables.pack_problem(*scenarios.scenario("cfg2"))
    tw = scenarios.trace_windows("cfg2")
    win = tables.window_arrays(tw["prefill_qps"][:24], tw["prefill_len"][:24], 0, 2.0)
    for mode in (abi.MODE_MODEL, abi.MODE_OPERATOR):
        prm = model.AutoscaleParams(slo=2.0)
        dec = _native.plan_windows_host(mode, prob, win, model=tables.pack_model(prob, prm),
                                        greedy=tables.pack_greedy(prob, prm))
        # per-window placement SLOs straddling the planning SLO (OPSC_PLACE_WINDOW_SLO)
        pwin = tables.window_arrays(tw["prefill_qps"][:24], tw["prefill_len"][:24], 0,
                                    np.linspace(1.2, 2.4, 24))
        for theta, caps in ((0.5, [80e9]), (1.5, [180e9, 40e9])):
            devs = [model.DeviceSpec(id=f"g{i:04d}", mem_cap=caps[i % len(caps)]) for i in range(2048)]
            for ds in (False, True):
                for wslo in (False, True):
                    fleet = placement.SharedFleet(devs, 2.0, model.InterferenceParams(theta, 1.0),
                                                  model.EnergyParams(), default_stream=ds, window_slo=wslo)
                    w = pwin if wslo else win
                    gpu = placement.place_windows(prob, w, dec.cfg, dec.feasible, fleet, 1)
                    cpu = orc.place_shared(prob, w, dec.cfg, dec.feasible, fleet, 1)
                    for f in placement.PlacementArrays.FIELDS:
                        assert getattr(gpu, f).tobytes() == getattr(cpu, f).tobytes(), (mode, theta, ds, wslo, f)


def test_place_dropin_matches_reference_objects():
    """placement.place() (reference signature) on GPU-decided plans returns
    the reference's Placement field for field (golden 'a100' setting)."""
    from paper_2511_02248_b200 import planners
    setting = next(s for s in TP.SETTINGS if s[0] == "a100")
    checked = 0
    for rec in TP.CASES[::5]:
        exp = rec["settings"]["a100"]
        src = G.load(rec["source"])
        c = next(c for c in src if c["name"] == rec["name"])
        dag_spec, prof = (scenarios.SCENARIOS[c["scenario"]] if "scenario" in c
                          else (c["dag"], c["profiles"]))
        dag, profiles = model.build_dag(dag_spec), model.profiles_from_dict(prof)
        params, pt = G.case_params(c), G.case_point(c)
        if rec["source"] == "oracle.json":
            plan = planners.brute_force_autoscale(dag, profiles, pt, params, G.case_bounds(c), guards=False)
        elif rec["source"] == "model.json":
            plan = planners.model_level_autoscale(dag, profiles, pt, params)
        else:
            plan = planners.greedy_autoscale(dag, profiles, pt, params)
        assert [[op, cf.p, cf.r, cf.b] for op, cf in plan.configs.items()] == rec["plan"]
        name, n, caps, ccap, theta, expo, over = setting
        width = len(str(max(0, n - 1)))
        fleet = [model.DeviceSpec(id=f"dev{i:0{width}d}", mem_cap=caps[i % len(caps)], compute_cap=ccap)
                 for i in range(n)]
        profiles.interference = model.InterferenceParams(theta, expo)
        pp = model.PlacementParams(slo=params.slo, **over)
        if "error" in exp:
            with pytest.raises(Exception) as ei:
                placement.place(plan, dag, profiles, fleet, pp, pt)
            assert type(ei.value).__name__ == exp["error"]
            continue
        placed, energy, memory = placement.place(plan, dag, profiles, fleet, pp, pt, return_metrics=True)
        got = [[a.op_id, a.replica_index, a.device_id, a.sm_share, a.interference_adjusted_latency.hex()]
               for a in placed.assignments]
        assert got == exp["assignments"], rec["name"]
        assert [[d, l.mem_used.hex(), l.sm_demand.hex(), l.energy.hex()]
                for d, l in placed.device_loads.items()] == exp["devices"]
        assert (placed.devices_used, placed.feasible, placed.recomputed_latency.hex()) == \
            (exp["devices_used"], exp["feasible"], exp["recomputed_latency"])
        assert (energy.hex(), memory.hex()) == (exp["energy"], exp["memory"])
        checked += 1
    assert checked > 10


def test_gpu_place_odd_workspace_strides(orc):
    """Odd assignment / device capacities (per-window workspace strides that
    are not multiples of 8 B before rounding) on many windows, incl.
    FleetExhausted mid-batch."""
    from paper_2511_02248_b200 import _native
    prob = tables.pack_problem(*scenarios.scenario("cfg1"))
    tw = scenarios.trace_windows("cfg2")
    win = tables.window_arrays(tw["prefill_qps"][:33] * 3.0, tw["prefill_len"][:33], 0, 0.5)
    prm = model.AutoscaleParams(slo=0.5)
    dec = _native.plan_windows_host(abi.MODE_OPERATOR, prob, win, model=tables.pack_model(prob, prm),
                                    greedy=tables.pack_greedy(prob, prm))
    for n_dev in (1, 3, 5, 7, 9, 31):
        devs = [model.DeviceSpec(id=f"d{i:02d}", mem_cap=80e9) for i in range(n_dev)]
        for ds in (False, True):
            fleet = placement.SharedFleet(devs, 0.5, model.InterferenceParams(0.5, 1.0), model.EnergyParams(),
                                          default_stream=ds)
            gpu = placement.place_windows(prob, win, dec.cfg, dec.feasible, fleet, 1)
            cpu = orc.place_shared(prob, win, dec.cfg, dec.feasible, fleet, 1)
            assert np.array_equal(gpu.status, cpu.status), n_dev
            bad = gpu.status != 0
            for f in placement.PlacementArrays.FIELDS:
                g, c = getattr(gpu, f).copy(), getattr(cpu, f).copy()
                g[bad] = 0  # a failed window's slots are unspecified (only status counts)
                c[bad] = 0
                assert g.tobytes() == c.tobytes(), (n_dev, ds, f)


@pytest.mark.parametrize("n_dev", [600, 4096])
def test_gpu_place_more_devices_than_a_probe_chunk(orc, n_dev):
    """Windows whose plans use more devices than one probe chunk holds
    (kMaxDevProbe = 128: the extras probe the fleet in chunks, the best score
    carried across them), with the per-window workspace in shared memory
    (600 devices) and in global memory (4096 devices), against the oracle."""
    from paper_2511_02248_b200 import _native
    prob = tables.pack_problem(*scenarios.scenario("cfg2"))
    tw = scenarios.trace_windows("cfg2")
    idx = np.argsort(tw["prefill_qps"])[-4:]
    win = tables.window_arrays(tw["prefill_qps"][idx] * 4.0, tw["prefill_len"][idx], 0, 2.0)
    prm = model.AutoscaleParams(slo=2.0)
    dec = _native.plan_windows_host(abi.MODE_OPERATOR, prob, win, model=tables.pack_model(prob, prm),
                                    greedy=tables.pack_greedy(prob, prm))
    devs = [model.DeviceSpec(id=f"g{i:04d}", mem_cap=80e9) for i in range(n_dev)]
    for ds in (False, True):
        fleet = placement.SharedFleet(devs, 2.0, model.InterferenceParams(0.5, 1.0), model.EnergyParams(),
                                      default_stream=ds)
        gpu = placement.place_windows(prob, win, dec.cfg, dec.feasible, fleet, 1)
        cpu = orc.place_shared(prob, win, dec.cfg, dec.feasible, fleet, 1)
        assert (cpu.status == 0).all() and cpu.devices_used.min() > 128
        for f in placement.PlacementArrays.FIELDS:
            assert getattr(gpu, f).tobytes() == getattr(cpu, f).tobytes(), (n_dev, ds, f)
