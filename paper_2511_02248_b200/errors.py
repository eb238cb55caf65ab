"""Exception taxonomy of the planner API this package stands in for.

Names and meanings follow the reference (errors.py:8-9 base class; concrete
errors next to the code that raises them: autoscaler.py:36-41,
perfmodel.py:33-46, opgraph.py:29-38, queueing.py:27-32, placement.py:38-43).
When the reference package is installed, `install.install()` maps raised
errors onto the reference's own classes instead.
"""


class OpscalerError(Exception):
    """Base class for all planner errors."""


class NoStableConfig(OpscalerError):
    """No (B, P, R <= r_cap) keeps an operator's queue stable."""


class SearchSpaceTooLarge(OpscalerError):
    """Brute-force enumeration would exceed the configured guard."""


class UnknownProfile(OpscalerError):
    """A profile_ref or volume_ref does not resolve in the ProfileSet."""


class UnknownPhase(OpscalerError):
    """Phase tag other than 'prefill' or 'decode', or a profile lacking it."""


class CycleDetected(OpscalerError):
    """The edge set admits no topological order."""


class DanglingEdge(OpscalerError):
    """An edge endpoint names a node that does not exist."""


class Unstable(OpscalerError):
    """Arrival rate meets or exceeds total service capacity (rho >= 1)."""


class FleetExhausted(OpscalerError):
    """No unused device remains for a replica that must be provisioned."""


class InfeasiblePlacement(OpscalerError):
    """A replica cannot be hosted on any device."""


class DeviceUnavailable(OpscalerError):
    """The CUDA extension is missing or no B200 is visible: there is no
    CPU fallback for the planner search."""


class MismatchedScenario(OpscalerError):
    """Savings comparison across different workload/SLO fingerprints
    (metrics.py:30-31)."""


class ParseError(OpscalerError):
    """Malformed trace file (workload.py:23-24)."""


class EmptyTrace(OpscalerError):
    """Trace file without data rows (workload.py:27-28)."""
