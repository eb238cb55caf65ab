"""Reroute an installed reference planner (`opscaler`) onto the GPU search.

The reference has no plugin registry: runner.plan_for_mode resolves
`autoscaler.greedy_autoscale / model_level_autoscale / brute_force_autoscale`
by module attribute at call time (runner.py:38-52), and the planners call
each other by global name inside autoscaler.py (:352, :497, :771). Rebinding
those module attributes therefore reroutes the CLI (all three --mode values),
runner.sweep / compare_point and the planners' internal calls without editing
the reference.

    import opscaler
    from paper_2511_02248_b200 import install
    install(opscaler)   # planners, placement, runner.sweep and cli.cmd_autoscale
                        # now run on the B200

The wrappers accept the reference's own objects, return the reference's own
ScalingPlan / OperatorConfig / PredictedSojourn instances and raise its own
exception classes. `MAX_ENUMERATION` is read from opscaler.autoscaler at call
time, as the reference does (autoscaler.py:735).
"""

from __future__ import annotations

import functools
import types

from . import planners


def _namespaces(pkg):
    A = pkg.autoscaler
    types_ns = types.SimpleNamespace(
        OperatorConfig=A.OperatorConfig, PredictedSojourn=A.PredictedSojourn,
        ScalingPlan=A.ScalingPlan, BruteForceBounds=A.BruteForceBounds)
    PL = pkg.placement
    types_ns.ReplicaAssignment = PL.ReplicaAssignment
    types_ns.DeviceLoad = PL.DeviceLoad
    types_ns.Placement = PL.Placement
    err_ns = types.SimpleNamespace(
        NoStableConfig=A.NoStableConfig, SearchSpaceTooLarge=A.SearchSpaceTooLarge,
        Unstable=pkg.queueing.Unstable, FleetExhausted=PL.FleetExhausted,
        InfeasiblePlacement=PL.InfeasiblePlacement)
    return types_ns, err_ns


def _runner_types(pkg, T, E):
    from . import runner as gpu_runner
    E.MismatchedScenario = pkg.metrics.MismatchedScenario

    class RT(gpu_runner.Types):
        PointResult = pkg.runner.PointResult
        ScenarioEval = pkg.metrics.ScenarioEval
        SavingsReport = pkg.metrics.SavingsReport
        ComparisonRow = pkg.runner.ComparisonRow
        plan_types = T
        err = E
    return RT


def install(pkg=None):
    """Rebind the reference's planners to the GPU drop-ins; returns an
    `uninstall` callable restoring the originals."""
    if pkg is None:
        import opscaler as pkg  # noqa: F811
    import importlib
    for sub in ("autoscaler", "placement", "runner", "cli", "metrics", "queueing"):
        importlib.import_module(f"{pkg.__name__}.{sub}")  # submodules the wrappers rebind
    A = pkg.autoscaler
    T, E = _namespaces(pkg)
    names = ("brute_force_autoscale", "model_level_autoscale", "greedy_autoscale")
    saved = {(mod, name): getattr(mod, name, None) for mod in (A, pkg) for name in names}
    saved[(pkg.placement, "place")] = pkg.placement.place
    saved[(pkg, "place")] = getattr(pkg, "place", None)

    @functools.wraps(saved[(A, "brute_force_autoscale")])
    def brute_force_autoscale(dag, profiles, point, params, bounds=None):
        return planners.brute_force_autoscale(
            dag, profiles, point, params, bounds, types=T, err=E,
            max_enumeration=A.MAX_ENUMERATION)

    @functools.wraps(saved[(A, "model_level_autoscale")])
    def model_level_autoscale(dag, profiles, point, params):
        return planners.model_level_autoscale(dag, profiles, point, params, types=T, err=E)

    @functools.wraps(saved[(A, "greedy_autoscale")])
    def greedy_autoscale(dag, profiles, point, params):
        return planners.greedy_autoscale(dag, profiles, point, params, types=T, err=E)

    from . import placement as gpu_placement

    @functools.wraps(saved[(pkg.placement, "place")])
    def place(plan, dag, profiles, fleet, params, point):
        return gpu_placement.place(plan, dag, profiles, fleet, params, point, types=T, err=E)

    for mod in (A, pkg):
        mod.brute_force_autoscale = brute_force_autoscale
        mod.model_level_autoscale = model_level_autoscale
        mod.greedy_autoscale = greedy_autoscale
    pkg.placement.place = place
    pkg.place = place

    @functools.wraps(pkg.placement.default_stream_place)
    def default_stream_place(plan, dag, profiles, fleet, params, point):
        return gpu_placement.default_stream_place(plan, dag, profiles, fleet, params, point,
                                                  types=T, err=E)

    saved[(pkg.placement, "default_stream_place")] = pkg.placement.default_stream_place
    pkg.placement.default_stream_place = default_stream_place

    # batched runner: sweep (runner.py:190-240) and cli.cmd_autoscale
    # (cli.py:123-186) plan and place all points of a DAG per launch
    from . import runner as gpu_runner
    RT = _runner_types(pkg, T, E)

    @functools.wraps(pkg.runner.sweep)
    def sweep(axis, values, dag, profiles, fleet, base_point, params, placement_mode="shared",
              energy_params=None, max_workers=4):
        return gpu_runner.sweep(axis, values, dag, profiles, fleet, base_point, params,
                                placement_mode, energy_params, max_workers, types=RT)

    cli = pkg.cli

    @functools.wraps(cli.cmd_autoscale)
    def cmd_autoscale(args):
        dag, profiles, fleet = cli._load_scenario(args)
        windows = cli._workload_points(args)
        return gpu_runner.autoscale_windows(dag, profiles, fleet, windows, args.mode, args.placement,
                                            lambda ph: cli._params(args, ph), args.out, types=RT,
                                            max_enumeration=A.MAX_ENUMERATION)

    for mod, name, fn in ((pkg.runner, "sweep", sweep), (cli, "cmd_autoscale", cmd_autoscale)):
        saved[(mod, name)] = getattr(mod, name)
        setattr(mod, name, fn)

    def uninstall():
        for (mod, name), fn in saved.items():
            if fn is not None:
                setattr(mod, name, fn)

    return uninstall
