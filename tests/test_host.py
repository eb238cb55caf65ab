"""Host-side logic: table packing, argument checks and error order of the
drop-in planners (all raised before any device work), the installer, and the
workload mirror against the reference-generated trace fixture."""

import contextlib
import io
import os
import sys
import tempfile

import numpy as np
import pytest

import golden_cases as G
from paper_2511_02248_b200 import (
    NoStableConfig, SearchSpaceTooLarge, UnknownPhase, UnknownProfile, abi, model, planners,
    tables, workload,
)
from workloads import scenarios


def test_pack_problem_topology():
    dag, prof = scenarios.scenario("cfg3")
    p = tables.pack_problem(dag, prof)
    assert p.ids == sorted(dag.node_ids)
    assert [p.ids[x] for x in p.table.topo[:p.n_ops]] == dag.topo_order
    assert [p.ids[x] for x in p.table.node_order[:p.n_ops]] == dag.node_ids
    for v, op in enumerate(p.ids):
        preds = {p.ids[u] for u in range(p.n_ops) if p.table.pred_mask[v] >> u & 1}
        assert preds == set(dag.predecessors(op))
        assert bool(p.table.sink_mask >> v & 1) == (not dag.successors(op))
        assert p.table.out_ptr[v + 1] - p.table.out_ptr[v] == len(dag.out_edges(op))
    # two sources merge into the LLM stack
    assert sorted(dag.sources) == ["embed", "patch_embed"]


def test_topo_order_matches_reference_rule():
    """Kahn with a sorted ready list (opgraph.py:110-132) on random DAGs."""
    rng = np.random.default_rng(5)
    for _ in range(50):
        n = int(rng.integers(2, 12))
        ids = [f"x{int(i)}" for i in rng.permutation(n)]
        edges = [{"src": ids[i], "dst": ids[j]} for j in range(n) for i in range(j)
                 if rng.uniform() < 0.3]
        dag = model.build_dag({"nodes": [{"id": i} for i in ids], "edges": edges})
        # reference rule, restated
        indeg = {i: 0 for i in ids}
        succ = {i: [] for i in ids}
        for e in edges:
            indeg[e["dst"]] += 1
            succ[e["src"]].append(e["dst"])
        ready, order = sorted(i for i in ids if indeg[i] == 0), []
        while ready:
            v = ready.pop(0)
            order.append(v)
            ins = False
            for w in sorted(succ[v]):
                indeg[w] -= 1
                if indeg[w] == 0:
                    ready.append(w)
                    ins = True
            if ins:
                ready.sort()
        assert dag.topo_order == order


def test_grid_menu_layout():
    dag, prof = scenarios.scenario("cfg5")
    p = tables.pack_problem(dag, prof)
    g = tables.pack_grid(p, model.AutoscaleParams(slo=0.5),
                         model.BruteForceBounds(r_max=4, b_max=3, parallelism=(2, 1)))
    assert tables.menu_sizes(p, g) == [24] * 6
    assert list(g.p_vals[0][:2]) == [1, 2]  # sorted, as bounds.parallelism_for sorts
    assert planners.candidate_space(p, g) == 24 ** 6


def _cfg1_point(qps=10.0):
    return model.WorkloadPoint(qps, 1024, "prefill")


def test_error_order_before_device():
    dag, prof = scenarios.scenario("cfg1")
    params = model.AutoscaleParams(slo=0.5)
    with pytest.raises(ValueError, match="qps > 0"):
        planners.brute_force_autoscale(dag, prof, model.WorkloadPoint(0.0, 10, "prefill"), params)
    with pytest.raises(SearchSpaceTooLarge, match="projected enumeration"):
        planners.brute_force_autoscale(dag, prof, _cfg1_point(), params,
                                       model.BruteForceBounds(r_max=8))
    big, bprof = scenarios.scenario("cfg2")
    with pytest.raises(SearchSpaceTooLarge, match="10 operators > 6"):
        planners.brute_force_autoscale(big, bprof, _cfg1_point(), params,
                                       model.BruteForceBounds(r_max=1, b_max=1, parallelism=(1,)))
    bad = dict(scenarios.PROFILES_7B)
    del bad["attn"]
    with pytest.raises(UnknownProfile):
        planners.brute_force_autoscale(dag, model.profiles_from_dict(bad), _cfg1_point(), params)
    nodecode = {k: ({kk: vv for kk, vv in v.items() if kk != "decode"} if isinstance(v, dict) and "prefill" in v else v)
                for k, v in scenarios.PROFILES_7B.items()}
    with pytest.raises(UnknownPhase):
        planners.model_level_autoscale(dag, model.profiles_from_dict(nodecode),
                                       model.WorkloadPoint(100.0, 1, "decode"), params)


def test_max_enumeration_is_read_at_call_time(monkeypatch):
    dag, prof = scenarios.scenario("cfg1")
    b = model.BruteForceBounds(r_max=3, b_max=2, parallelism=(1, 2))  # 12^6 ~ 3e6
    monkeypatch.setattr(planners, "MAX_ENUMERATION", 1000)
    with pytest.raises(SearchSpaceTooLarge):
        planners.brute_force_autoscale(dag, prof, _cfg1_point(), model.AutoscaleParams(slo=0.5), b)


def test_status_to_exception_mapping():
    from paper_2511_02248_b200 import plans
    with pytest.raises(NoStableConfig):
        plans.raise_for_status(abi.W_NO_STABLE_PARAMS, abi.MODE_ORACLE)
    with pytest.raises(NoStableConfig):
        plans.raise_for_status(abi.W_NO_STABLE_BOUNDS, abi.MODE_ORACLE)
    with pytest.raises(NoStableConfig):
        plans.raise_for_status(abi.W_NO_STABLE_MODEL, abi.MODE_MODEL)
    with pytest.raises(ZeroDivisionError):
        plans.raise_for_status(abi.W_ZERO_DIVISION | abi.W_NO_STABLE_PARAMS, abi.MODE_ORACLE)
    plans.raise_for_status(abi.W_FLEET_EXHAUSTED, abi.MODE_ORACLE)  # placement is not a planner error


def test_plan_materialisation_from_arrays(orc):
    """WindowDecisions builds reference-shaped plans (oracle arrays here)."""
    from paper_2511_02248_b200 import plans
    c = next(c for c in G.load("oracle.json") if c["name"] == "cfg1/w0/prefill")
    prob = G.case_problem(c)
    win = G.case_windows(c)
    out = orc.plan_windows(abi.MODE_ORACLE, prob, win,
                           grid=tables.pack_grid(prob, G.case_params(c), G.case_bounds(c)))
    plan = plans.WindowDecisions(prob, [G.case_point(c)], out, abi.MODE_ORACLE).plan(0)
    assert plan.to_dict()["operators"] == {op: {"P": p, "R": r, "B": b, "sm_share": 100}
                                           for op, p, r, b in c["expected"]["configs"]}


REF = "/root/reference/pkg/src"


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference not present (GPU box)")
def test_installer_reroutes_reference():
    sys.path.insert(0, REF)
    try:
        import opscaler
        from opscaler import runner
        from paper_2511_02248_b200 import DeviceUnavailable, install, _native
        orig = opscaler.autoscaler.brute_force_autoscale
        from opscaler import cli
        orig_cli = (cli.cmd_autoscale, runner.sweep, opscaler.placement.default_stream_place)
        undo = install(opscaler)
        try:
            assert opscaler.autoscaler.brute_force_autoscale is not orig
            dag = opscaler.build_dag(scenarios.DAG_70B)
            prof = opscaler.perfmodel.profiles_from_dict(scenarios.PROFILES_70B)
            pt = opscaler.WorkloadPoint(10.0, 512, "prefill")
            params = opscaler.AutoscaleParams(slo=1.0)
            # the reference's own guard exception class, raised by our wrapper
            with pytest.raises(opscaler.autoscaler.SearchSpaceTooLarge):
                runner.plan_for_mode("oracle", dag, prof, pt, params,
                                     opscaler.BruteForceBounds(r_max=1, b_max=1))
            if _native.device_count() == 0:
                with pytest.raises(DeviceUnavailable):
                    runner.plan_for_mode("model", dag, prof, pt, params)
            # the CLI: cmd_autoscale and runner.sweep are the batched drop-ins
            now = (cli.cmd_autoscale, runner.sweep, opscaler.placement.default_stream_place)
            assert all(a is not b for a, b in zip(now, orig_cli))
            import golden_cases as G
            gdir = os.path.join(os.path.dirname(__file__), "golden", "cli")
            cwd = os.getcwd()
            os.chdir(gdir)
            try:
                for c in G.load("cli.json"):
                    if c["name"] == "auto_7b_oracle_guard":
                        err = io.StringIO()
                        with contextlib.redirect_stderr(err):
                            assert cli.main(c["argv"] + ["--out", tempfile.mkdtemp()]) == c["exit"]
                        assert err.getvalue() == c["stderr"]
                    elif c["name"] == "sweep_qps" and _native.device_count() == 0:
                        with pytest.raises(DeviceUnavailable):
                            cli.main(c["argv"] + ["--out", tempfile.mkdtemp()])
            finally:
                os.chdir(cwd)
        finally:
            undo()
        assert opscaler.autoscaler.brute_force_autoscale is orig
        assert (cli.cmd_autoscale, runner.sweep, opscaler.placement.default_stream_place) == orig_cli
    finally:
        sys.path.remove(REF)


@pytest.mark.parametrize("cfg", ["cfg1", "cfg2", "cfg3"])
def test_workload_mirror_matches_reference_fixture(cfg):
    spec = scenarios.TRACES[cfg]
    recs = workload.synth_workload(workload.SynthSpec(**spec["spec"]), spec["seed"])
    wins = workload.windowize(recs, spec["window_len"], spec["quantile"])
    tw = scenarios.trace_windows(cfg)
    head = np.array([(r.arrival_time, r.input_len, r.output_len) for r in recs[:5000]])
    assert np.array_equal(head, tw["head_records"])
    assert np.array_equal(np.array([p.qps for p, _ in wins]), tw["prefill_qps"])
    assert np.array_equal(np.array([p.seq_len for p, _ in wins]), tw["prefill_len"])
    assert np.array_equal(np.array([d.qps for _, d in wins]), tw["decode_qps"])


@pytest.mark.parametrize("cfg", ["cfg1", "cfg2", "cfg3", "cfg5"])
def test_oracle_windowize_matches_reference_fixture(orc, cfg):
    spec = scenarios.TRACES[cfg]
    recs = workload.synth_workload(workload.SynthSpec(**spec["spec"]), spec["seed"])
    arr = np.array([r.arrival_time for r in recs])
    li = np.array([r.input_len for r in recs])
    lo = np.array([r.output_len for r in recs])
    pq, pl, dq = orc.windowize(arr, li, lo, spec["window_len"], spec["quantile"])
    tw = scenarios.trace_windows(cfg)
    assert np.array_equal(pq, tw["prefill_qps"])
    assert np.array_equal(pl, tw["prefill_len"])
    assert np.array_equal(dq, tw["decode_qps"])
    # order independence (windowize buckets; the quantile sorts)
    perm = np.random.default_rng(0).permutation(len(arr))
    pq2, pl2, dq2 = orc.windowize(arr[perm], li[perm], lo[perm], spec["window_len"], spec["quantile"])
    assert np.array_equal(pq, pq2) and np.array_equal(pl, pl2) and np.array_equal(dq, dq2)


def test_error_texts_match_reference(orc):
    from paper_2511_02248_b200 import errors, plans
    """NoStableConfig raised from device status words carries the reference's
    own text (operator named via the status op fields): init_configs
    (autoscaler.py:289-292) in oracle and greedy mode, the bounds fallback
    (:835-837), model level (:678-681). Decisions come from the CPU oracle
    here (same status words as the kernels, checked bitwise on the GPU)."""
    import refpkg
    op = refpkg.import_reference()
    dag_spec, prof = scenarios.SCENARIOS["cfg1"]
    rdag, rprof = op.build_dag(dag_spec), op.perfmodel.profiles_from_dict(prof)
    dag, profm = model.build_dag(dag_spec), model.profiles_from_dict(prof)
    prob = tables.pack_problem(dag, profm)
    cases = [("oracle", dict(qps=1e9, seq_len=2048), dict(slo=0.5), dict(r_max=3, b_max=2, parallelism=(1, 2))),
             ("oracle", dict(qps=40.0, seq_len=4096), dict(slo=0.5), dict(r_max=1, b_max=1, parallelism=(1,))),
             ("operator", dict(qps=1e9, seq_len=2048), dict(slo=0.5), None),
             ("operator", dict(qps=3e4, seq_len=2048), dict(slo=0.5, r_cap=64), None),   # attn
             ("oracle", dict(qps=1e5, seq_len=2048), dict(slo=0.5, r_cap=16),            # qkv
              dict(r_max=3, b_max=2, parallelism=(1, 2))),
             ("model", dict(qps=5e4, seq_len=2048), dict(slo=0.5, r_cap=4), None)]
    seen = 0
    for mode, pt, prm, bnd in cases:
        rpt = op.WorkloadPoint(pt["qps"], pt["seq_len"], "prefill")
        rparams = op.AutoscaleParams(**prm)
        with pytest.raises(op.autoscaler.NoStableConfig) as want:
            op.runner.plan_for_mode(mode, rdag, rprof, rpt, rparams,
                                    op.BruteForceBounds(**bnd) if bnd else None)
        mpt = model.WorkloadPoint(pt["qps"], pt["seq_len"], "prefill")
        params = model.AutoscaleParams(**prm)
        m = {"oracle": abi.MODE_ORACLE, "model": abi.MODE_MODEL, "operator": abi.MODE_OPERATOR}[mode]
        win = tables.pack_windows([mpt], params.slo, params.epsilon)
        out = orc.plan_windows(m, prob, win,
                               grid=tables.pack_grid(prob, params, model.BruteForceBounds(**bnd)) if bnd else None,
                               model=tables.pack_model(prob, params), greedy=tables.pack_greedy(prob, params))
        dec = plans.WindowDecisions(prob, [mpt], out, m, r_cap=params.r_cap)
        with pytest.raises(errors.NoStableConfig) as got:
            dec.plan(0)
        assert str(got.value) == str(want.value), mode
        seen += 1
    assert seen == len(cases)


@pytest.mark.parametrize("qps", [float("nan"), float("inf")])
def test_nonfinite_qps_raises_like_reference(orc, qps):
    """NaN / +inf qps pass the reference's `qps <= 0` check and fail in
    _strict_min_replicas (autoscaler.py:225) in every planner: same class and
    text from the drop-in (the device treats the window as idle)."""
    from paper_2511_02248_b200 import plans
    import refpkg
    op = refpkg.import_reference()
    dag_spec, prof = scenarios.SCENARIOS["cfg1"]
    rdag, rprof = op.build_dag(dag_spec), op.perfmodel.profiles_from_dict(prof)
    prob = tables.pack_problem(model.build_dag(dag_spec), model.profiles_from_dict(prof))
    for mode, m in (("oracle", abi.MODE_ORACLE), ("model", abi.MODE_MODEL), ("operator", abi.MODE_OPERATOR)):
        bnd = dict(r_max=2, b_max=1, parallelism=(1,))
        with pytest.raises(Exception) as want:
            op.runner.plan_for_mode(mode, rdag, rprof, op.WorkloadPoint(qps, 512, "prefill"),
                                    op.AutoscaleParams(slo=0.5), op.BruteForceBounds(**bnd))
        pt = model.WorkloadPoint(qps, 512, "prefill")
        params = model.AutoscaleParams(slo=0.5)
        out = orc.plan_windows(m, prob, tables.pack_windows([pt], 0.5, 0.0),
                               grid=tables.pack_grid(prob, params, model.BruteForceBounds(**bnd)),
                               model=tables.pack_model(prob, params), greedy=tables.pack_greedy(prob, params))
        with pytest.raises(Exception) as got:
            plans.WindowDecisions(prob, [pt], out, m, r_cap=512).plan(0)
        assert type(got.value) is type(want.value) and str(got.value) == str(want.value), mode
