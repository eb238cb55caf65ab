"""§8(f) row 4: the batched runner / CLI reproduces the reference CLI's
artifacts byte for byte (plan_*.json, placement_*.json, metrics.csv,
sweep_*.csv), exit codes and error text (tests/golden/cli.json)."""

import contextlib
import hashlib
import io
import os
import tempfile

import pytest

import golden_cases as G
from paper_2511_02248_b200 import cli

pytestmark = pytest.mark.gpu

IN = os.path.join(os.path.dirname(__file__), "golden", "cli")
CASES = G.load("cli.json")


def run_case(argv):
    with tempfile.TemporaryDirectory() as tmp:
        out = os.path.join(tmp, "out")
        err = io.StringIO()
        cwd = os.getcwd()
        os.chdir(IN)
        try:
            with contextlib.redirect_stderr(err):
                rc = cli.main(argv + ["--out", out])
        finally:
            os.chdir(cwd)
        files = {}
        if os.path.isdir(out):
            for name in sorted(os.listdir(out)):
                with open(os.path.join(out, name), "rb") as fh:
                    files[name] = fh.read()
        return rc, err.getvalue(), files


@pytest.mark.parametrize("case", CASES, ids=lambda c: c["name"])
def test_cli_artifacts_byte_identical(case):
    rc, err, files = run_case(case["argv"])
    for name, text in case["texts"].items():
        assert files.get(name, b"").decode() == text, name
    got = {k: hashlib.sha256(v).hexdigest() for k, v in files.items()}
    bad = [k for k in case["files"] if got.get(k) != case["files"][k]]
    assert not bad, (bad[:3], files.get(bad[0], b"")[:400])
    assert sorted(got) == sorted(case["files"])
    assert rc == case["exit"]
    assert err == case["stderr"]
