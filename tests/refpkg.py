"""Locate the UNMODIFIED reference package (`opscaler`) for drop-in tests.

TEST INFRASTRUCTURE. On the GPU box the reference is the copy installed by
`python -m pip install --no-index --no-build-isolation --no-deps --target
baseline/_ref <copy of /root/reference>/pkg` (git-ignored, travels with the
gpurun snapshot); in the build container /root/reference/pkg/src is used
directly. Tests that need it skip when neither exists. The product package
never imports the reference.
"""

import importlib
import os
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CANDIDATES = (os.path.join(REPO, "baseline", "_ref"), "/root/reference/pkg/src")


def path():
    for p in CANDIDATES:
        if os.path.isfile(os.path.join(p, "opscaler", "__init__.py")):
            return p
    return None


def import_reference():
    if "opscaler" in sys.modules:  # already imported (by another test) from a candidate path
        mod = sys.modules["opscaler"]
        assert os.path.dirname(os.path.dirname(mod.__file__)) in CANDIDATES, mod.__file__
        for sub in ("runner", "cli"):
            importlib.import_module("opscaler." + sub)
        return mod
    p = path()
    if p is None:
        pytest.skip("reference package not installed (baseline/_ref) and /root/reference absent")
    if p not in sys.path:
        sys.path.insert(0, p)
    mod = importlib.import_module("opscaler")
    for sub in ("runner", "cli"):  # not imported by the package __init__
        importlib.import_module("opscaler." + sub)
    assert os.path.dirname(os.path.dirname(mod.__file__)) == p, mod.__file__
    return mod
