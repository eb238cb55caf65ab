"""The small-batch model-level path (every (B, R) point tabulated in parallel,
probe/bisect over the table) is bit-identical to the per-window probe path."""

import numpy as np
import pytest

from paper_2511_02248_b200 import abi, device, model, tables
from workloads import scenarios

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("cfg", ["cfg1", "cfg2", "cfg3"])
def test_table_path_equals_probe_path(cfg):
    prob = tables.pack_problem(*scenarios.scenario(cfg))
    tw = scenarios.trace_windows(cfg)
    for phase in ("prefill", "decode"):
        for eps in (0.0, 0.07):
            slo = scenarios.SLO[cfg][phase]
            prm = model.AutoscaleParams(slo=slo, epsilon=slo * eps)
            spec = tables.pack_model(prob, prm)
            win = tables.window_arrays(tw[phase + "_qps"][:4], tw[phase + "_len"][:4],
                                       tables.PHASE_INDEX[phase], slo, slo * eps)
            a = device.DevicePlanner(prob, win, abi.MODE_MODEL, model=spec)
            a.MODEL_TABLE_POINTS = 1 << 30  # force the table
            a.step()
            b = device.DevicePlanner(prob, win, abi.MODE_MODEL, model=spec)
            b.MODEL_TABLE_POINTS = 0        # force per-window probes
            b.step()
            da, db = a.decisions(), b.decisions()
            for f in tables.DecisionArrays.FIELDS:
                assert getattr(da, f).tobytes() == getattr(db, f).tobytes(), (cfg, phase, f)
