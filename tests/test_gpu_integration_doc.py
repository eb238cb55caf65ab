"""The ctypes binding shown in INTEGRATION.md §2 runs as written: the code
block is extracted from the document and executed against the built library
on the cfg1 DAG; its decisions equal the package's own host-buffer call."""

import os
import re

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)


def _snippet():
    text = open(os.path.join(REPO, "INTEGRATION.md")).read()
    sec = text[text.index("## 2. The C ABI and its ctypes binding"):]
    return re.search(r"```python\n(.*?)```", sec, re.S).group(1)


def test_integration_ctypes_snippet_runs():
    from paper_2511_02248_b200 import _native, abi, model, tables
    from workloads import scenarios
    dag, profiles = scenarios.scenario("cfg1")
    tw = scenarios.trace_windows("cfg1")
    params = model.AutoscaleParams(slo=scenarios.SLO["cfg1"]["prefill"])
    bounds = model.BruteForceBounds(**scenarios.GRIDS["cfg1"])
    points = [model.WorkloadPoint(float(tw["prefill_qps"][0]), int(tw["prefill_len"][0]), "prefill")]
    fleet, energy_params = None, None
    ns = dict(dag=dag, profiles=profiles, params=params, bounds=bounds, points=points, fleet=fleet,
              energy_params=energy_params)
    cwd = os.getcwd()
    os.chdir(REPO)  # the snippet loads the library by its repo-relative path
    try:
        exec(_snippet(), ns)  # noqa: S102 -- the document's own example
    finally:
        os.chdir(cwd)
    assert ns["rc"] == 0
    out = ns["out"]
    prob = tables.pack_problem(dag, profiles)
    want = _native.plan_windows_host(abi.MODE_ORACLE, prob, tables.pack_windows(points, params.slo, params.epsilon),
                                     grid=tables.pack_grid(prob, params, bounds))
    for f in tables.DecisionArrays.FIELDS:
        assert np.asarray(getattr(out, f)).tobytes() == np.asarray(getattr(want, f)).tobytes(), f
