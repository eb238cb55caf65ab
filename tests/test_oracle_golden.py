"""Pin the CPU restatement (oracle/) against the reference's own outputs.

Every vector in tests/golden/ was produced by running /root/reference
(tests/golden/make_golden.py); comparisons are bit-exact (float.hex).
"""

import ctypes as C
import json
import math

import numpy as np
import pytest

import golden_cases as G
from paper_2511_02248_b200 import abi, model, plans, tables


def test_erlang_c_kat(orc):
    for R, rho, exp in G.load("kats.json")["erlang_c"]:
        assert orc.lib().orc_erlang_c(R, G.F(rho)).hex() == exp, (R, rho)


def test_expected_wait_kat(orc):
    for lam, mu, R, exp in G.load("kats.json")["expected_wait"]:
        assert orc.lib().orc_expected_wait(G.F(lam), G.F(mu), R).hex() == exp


def test_spec_examples(orc):
    L = orc.lib()
    # SPEC.md:215-216, 224-226, 233-235
    assert L.orc_erlang_c(1, 0.5) == 0.5
    assert L.orc_erlang_c(2, 0.5) == 0.33333333333333337
    assert L.orc_expected_wait(1.0, 2.0, 1) == 0.5
    assert L.orc_strict_min_replicas(10.0, 3.0, 512) == 4
    assert L.orc_strict_min_replicas(6.0, 3.0, 512) == 3
    assert L.orc_strict_min_replicas(0.1, 100.0, 512) == 1
    # SPEC.md:132 (eta = 1)
    assert abs(L.orc_op_latency(0.0, 0.0, 1e-9, 1.0, 1, 2048, 1) - 4.194304e-3) < 1e-15
    # SPEC.md:141-142, 150
    assert L.orc_op_memory(16e9, 0.0, 0.0, 1, 1, 2) == 8e9
    assert L.orc_op_memory(0.0, 0.0, 2e4, 4, 1000, 1) == 8e7
    assert abs(L.orc_comm_time(0.0, 4096.0, 1, 1024, 600e9) - 6.99e-6) < 1e-8


def test_min_replicas_kat(orc):
    for lam, mu, mrs, strict in G.load("kats.json")["min_replicas_stable"]:
        got = orc.lib().orc_strict_min_replicas(G.F(lam), G.F(mu), 512)
        assert got == (strict if strict is not None else -1)
        assert orc.lib().orc_strict_min_replicas(G.F(lam), G.F(mu), 1 << 30) == mrs


def test_perfmodel_kat(orc):
    k = G.load("kats.json")
    L = orc.lib()
    for c, eta, B, Ln, P, exp in k["op_latency"]:
        got = L.orc_op_latency(G.F(c[0]), G.F(c[1]), G.F(c[2]), G.F(eta), B, Ln, P)
        assert got.hex() == exp
    for v0, v1, B, Ln, bw, exp in k["comm_time"]:
        assert L.orc_comm_time(G.F(v0), G.F(v1), B, Ln, G.F(bw)).hex() == exp
    for w, m0, m1, B, Ln, P, exp in k["op_memory"]:
        assert L.orc_op_memory(G.F(w), G.F(m0), G.F(m1), B, Ln, P).hex() == exp


def test_python_sum_emulation(orc):
    rng = np.random.default_rng(3)
    for _ in range(2000):
        xs = rng.uniform(0, 1, int(rng.integers(1, 14))) * 10 ** rng.uniform(-8, 11, 1)
        xs = np.ascontiguousarray(xs)
        assert orc.lib().orc_py_sum(xs.ctypes.data, len(xs)) == sum(xs.tolist())


def test_critical_path_kat(orc):
    for case in G.load("kats.json")["critical_path"]:
        dag = model.build_dag(case["dag"])
        prof = model.profiles_from_dict({n["id"]: {"prefill": {}} for n in case["dag"]["nodes"]})
        for n in dag.nodes:  # profile_ref defaults to the id
            assert n.profile_ref == n.id
        prob = tables.pack_problem(dag, prof)
        w = np.zeros(prob.n_ops)
        for op, (s, c) in case["sojourn"].items():
            w[prob.rank[op]] = (G.F(s) + G.F(c)) * dag.node(op).layer_count
        path = np.full(prob.n_ops, -1, dtype=np.int8)
        lat = orc.lib().orc_critical_path(orc.ref(prob.table), w.ctypes.data, path.ctypes.data)
        assert lat.hex() == case["latency"]
        assert [prob.ids[x] for x in path if x >= 0] == case["path"]


def test_menus_bit_exact(orc):
    for m in G.load("menus.json"):
        prob = G.case_problem(m)
        g = m["grid"]
        params = model.AutoscaleParams(slo=1.0)
        bounds = model.BruteForceBounds(r_max=g["r_max"], b_max=g["b_max"],
                                        parallelism=tuple(g["parallelism"]))
        grid = tables.pack_grid(prob, params, bounds)
        win = tables.pack_windows([G.case_point(m)], 1.0, 0.0)
        mw, st = orc.menus(prob, grid, win)
        assert st[0] == 0
        for op, rows in m["entries"].items():
            v = prob.rank[op]
            for e, row in enumerate(rows):
                assert mw[0, grid.menu_off[v] + e].hex() == row[6], (op, e, row)
                out = np.zeros(7)
                orc.lib().orc_predict(orc.ref(prob.table), win.qps[0], int(win.seq_len[0]),
                                      int(win.phase[0]), v, row[0], row[1], row[2],
                                      out.ctypes.data, None)
                assert [out[0].hex(), out[4].hex(), out[6].hex()] == row[3:6]


def _check_case(orc, c, mode):
    prob = G.case_problem(c)
    params = G.case_params(c)
    win = G.case_windows(c)
    grid = model_spec = None
    if mode == abi.MODE_ORACLE:
        grid = tables.pack_grid(prob, params, G.case_bounds(c))
    else:
        model_spec = tables.pack_model(prob, params)
    kinds = ["metrics", "metrics_small_fleet", "metrics_tiny_cap"] if mode == abi.MODE_ORACLE \
        else ["model_metrics"]
    errs = []
    for kind in kinds:
        place = tables.pack_place(G.fleet_for(kind), model.EnergyParams())
        out = orc.plan_windows(mode, prob, win, grid=grid, model=model_spec, place=place)
        dec = plans.WindowDecisions(prob, [G.case_point(c)], out, mode)
        exp = c["expected"]
        if "error" in exp:
            with pytest.raises(Exception) as ei:
                dec.plan(0)
            assert type(ei.value).__name__ == exp["error"]
            return
        if kind == kinds[0]:
            errs += G.compare_plan(dec.plan(0), exp, prob)
        golden_key = "metrics" if kind == "model_metrics" else kind
        errs += [f"{kind}: {e}" for e in G.compare_metrics(dec.metrics(0), c.get(golden_key))]
    assert not errs, (c["name"], errs)


@pytest.mark.parametrize("idx", range(len(G.load("oracle.json"))))
def test_oracle_decisions(orc, idx):
    c = G.load("oracle.json")[idx]
    _check_case(orc, c, abi.MODE_ORACLE)


@pytest.mark.parametrize("idx", range(len(G.load("model.json"))))
def test_model_decisions(orc, idx):
    c = G.load("model.json")[idx]
    _check_case(orc, c, abi.MODE_MODEL)


def _gt6_sample():
    """>6-op reference decisions (tests/golden/make_golden_gt6.py: the
    reference brute force with only its 6-op guard removed). The CPU oracle
    enumerates literally, so the suite checks every 6th cfg2 case (6^10 = 6e7
    candidates) and every 72nd cfg3 case (6^12 = 2.2e9); the GPU test checks
    all of them."""
    cs = G.load("oracle_gt6.json")
    idx = [i for i, c in enumerate(cs) if c["scenario"] == "cfg2"][::6]
    idx += [i for i, c in enumerate(cs) if c["scenario"] == "cfg3"][5::72]
    return idx


@pytest.mark.parametrize("idx", _gt6_sample())
def test_oracle_gt6_decisions(orc, idx):
    c = G.load("oracle_gt6.json")[idx]
    assert not c["hash_sensitive"]
    _check_case(orc, c, abi.MODE_ORACLE)


def test_gt6_golden_coverage():
    """The >6-op goldens exercise feasible winners, infeasible fallbacks and
    NoStableConfig on both DAGs and phases, with many distinct winners."""
    cs = G.load("oracle_gt6.json")
    for cfg in ("cfg2", "cfg3"):
        for ph in ("prefill", "decode"):
            sub = [c["expected"] for c in cs if c["scenario"] == cfg and c["point"]["phase"] == ph]
            feas = [e for e in sub if e.get("feasible")]
            assert len(feas) >= len(sub) // 3, (cfg, ph, len(feas), len(sub))
            assert len({json.dumps(e["configs"]) for e in feas}) >= 5, (cfg, ph)
    exp = [c["expected"] for c in cs]
    assert any("error" in e for e in exp)
    assert any(e.get("feasible") is False for e in exp)
    # the config SLO itself: most cfg2 windows have a feasible winner
    cfg2 = [c["expected"] for c in cs if c["scenario"] == "cfg2" and c["name"].endswith("slo_x1")]
    assert sum(bool(e.get("feasible")) for e in cfg2) >= 0.75 * len(cfg2)


def _check_greedy(orc, c):
    prob = G.case_problem(c)
    params = G.case_params(c)
    win = G.case_windows(c)
    place = tables.pack_place(G.fleet_for("model_metrics"), model.EnergyParams())
    out = orc.plan_windows(abi.MODE_OPERATOR, prob, win, greedy=tables.pack_greedy(prob, params),
                           place=place)
    dec = plans.WindowDecisions(prob, [G.case_point(c)], out, abi.MODE_OPERATOR)
    exp = c["expected"]
    if "error" in exp:
        with pytest.raises(Exception) as ei:
            dec.plan(0)
        assert type(ei.value).__name__ == exp["error"]
        return
    errs = G.compare_plan(dec.plan(0), exp, prob)
    errs += G.compare_metrics(dec.metrics(0), c.get("metrics"))
    assert not errs, (c["name"], errs)


@pytest.mark.parametrize("idx", range(len(G.load("greedy.json"))))
def test_greedy_decisions(orc, idx):
    _check_greedy(orc, G.load("greedy.json")[idx])


# tests/golden/make_golden_edges.py: slo = +inf (unstable, INF-weighted
# entries must stay out of the feasible set in every mode) and brute-force
# menus too large for the GPU's shared-memory tile
@pytest.mark.parametrize("fname,mode", [("edges_oracle.json", abi.MODE_ORACLE), ("edges_model.json", abi.MODE_MODEL),
                                        ("edges_greedy.json", abi.MODE_OPERATOR)])
def test_edge_decisions(orc, fname, mode):
    for c in G.load(fname):
        if mode == abi.MODE_OPERATOR:
            _check_greedy(orc, c)
        else:
            _check_case(orc, c, mode)
