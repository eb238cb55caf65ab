"""B200-native candidate-evaluation path of the opscaler planners
(arXiv 2511.02248 operator-level autoscaler).

Public surface (names and semantics of the reference's planner API,
pkg/src/opscaler/__init__.py:12-70):

  brute_force_autoscale, model_level_autoscale  -- drop-in planners (GPU)
  plan_windows, decide_windows                  -- batched per-window entry
  install                                       -- reroute an installed
                                                   `opscaler` to this path
  OperatorDag, ProfileSet, WorkloadPoint, AutoscaleParams, BruteForceBounds,
  OperatorConfig, PredictedSojourn, ScalingPlan, ... -- host data model

The search itself runs only on the CUDA extension (csrc/); there is no CPU
fallback. Importing this package does not load the extension; the first
planner call does, and raises DeviceUnavailable if it cannot.
"""

from .errors import (  # noqa: F401
    DeviceUnavailable, NoStableConfig, OpscalerError, SearchSpaceTooLarge,
    UnknownPhase, UnknownProfile,
)
from .model import (  # noqa: F401
    AutoscaleParams, BruteForceBounds, DeviceSpec, Edge, EnergyParams, LatencyModel,
    OperatorConfig, OperatorDag, OperatorNode, OperatorProfile, PredictedSojourn,
    ProfileSet, ScalingPlan, WorkloadPoint, build_dag, make_fleet, profiles_from_dict,
)

__version__ = "0.1.0"


def __getattr__(name):
    # planners pull in the native loader; keep package import CPU-safe
    if name in ("brute_force_autoscale", "model_level_autoscale", "greedy_autoscale", "plan_windows",
                "decide_windows", "MAX_ENUMERATION"):
        from . import planners
        return getattr(planners, name)
    if name == "install":
        from .installer import install
        return install
    raise AttributeError(name)
