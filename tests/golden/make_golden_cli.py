"""Freeze the reference CLI's artifacts.

Build container only (imports /root/reference). Writes the scenario inputs
(DAG / profile / fleet JSON, a trace CSV) under tests/golden/cli/, runs the
reference's own `opscaler` CLI (cli.main, cli.py:299-313) on each case into a
scratch directory and stores, per case, the exit code, the stderr text, the
sha256 of every output file and the full text of the CSVs, in
tests/golden/cli.json. tests/test_gpu_cli.py re-runs every case through
paper_2511_02248_b200.cli and requires byte-identical files.

    PYTHONHASHSEED=0 PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_cli.py
"""

import contextlib
import hashlib
import io
import json
import os
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, "/root/reference/pkg/src")

from opscaler import cli as ref_cli  # noqa: E402
from opscaler import workload as ref_workload  # noqa: E402

from workloads import scenarios  # noqa: E402

IN = os.path.join(HERE, "cli")

TINY_DAG = {"nodes": [{"id": "embed", "kind": "embedding", "layer_count": 1, "profile_ref": "embed"},
                      {"id": "mlp", "kind": "linear", "layer_count": 32, "profile_ref": "mlp"}],
            "edges": [{"src": "embed", "dst": "mlp", "volume_ref": "embed"}]}


def write_inputs():
    os.makedirs(IN, exist_ok=True)
    files = {
        "dag_7b.json": scenarios.DAG_7B, "profiles_7b.json": scenarios.PROFILES_7B,
        "dag_70b.json": scenarios.DAG_70B, "profiles_70b.json": scenarios.PROFILES_70B,
        "dag_mm.json": scenarios.DAG_MM, "profiles_mm.json": scenarios.PROFILES_MM,
        "dag_tiny.json": TINY_DAG,
        "fleet_64.json": [{"id": f"gpu{i:02d}", "mem_cap": 80e9} for i in range(64)],
        "fleet_4.json": [{"id": f"gpu{i}", "mem_cap": 80e9} for i in range(4)],
        "fleet_hetero.json": [{"id": f"node{(i * 7) % 96:02d}", "mem_cap": [80e9, 40e9, 180e9][i % 3],
                               "compute_cap": [1.0, 0.8, 1.3][i % 3]} for i in range(96)],
        "fleet_1k.json": [{"id": f"b200-{i:04d}", "mem_cap": 180e9} for i in range(1024)],
    }
    for name, obj in files.items():
        with open(os.path.join(IN, name), "w") as fh:
            json.dump(obj, fh, indent=1, sort_keys=True)
    # a trace with an idle gap (windows 3-4 empty) and unsorted rows
    recs = ref_workload.synth_workload(ref_workload.SynthSpec(kind="burst", rate=4.0, duration=420.0,
                                                              burst_factor=3.0, burst_duty=0.3,
                                                              input_len_median=2048.0), 3)
    recs = [r for r in recs if not (180.0 <= r.arrival_time < 300.0)]
    recs = recs[1::2] + recs[0::2]
    with open(os.path.join(IN, "trace_gap.csv"), "w") as fh:
        fh.write("timestamp_s,input_tokens,output_tokens\n")
        for r in recs:
            fh.write(f"{r.arrival_time!r},{r.input_len},{r.output_len}\n")


def scen(name, fleet):
    return ["--dag", f"dag_{name}.json", "--profiles", f"profiles_{name if name != 'tiny' else '7b'}.json",
            "--fleet", f"fleet_{fleet}.json"]


BURST = "burst:rate=8,duration=600,burst_factor=4,burst_duty=0.2,input_sigma=0.8"
CASES = [
    ("auto_7b_operator_shared", ["autoscale", *scen("7b", "64"), "--synth", BURST, "--mode", "operator"]),
    ("auto_7b_operator_default", ["autoscale", *scen("7b", "64"), "--synth", BURST, "--mode", "operator",
                                  "--placement", "default_stream"]),
    ("auto_7b_model_shared", ["autoscale", *scen("7b", "64"), "--synth", BURST, "--mode", "model"]),
    ("auto_7b_model_default", ["autoscale", *scen("7b", "64"), "--synth", BURST, "--mode", "model",
                               "--placement", "default_stream"]),
    ("auto_7b_eps", ["autoscale", *scen("7b", "64"), "--synth", BURST, "--mode", "operator",
                     "--epsilon", "0.01", "--slo-prefill", "0.4", "--slo-decode", "0.04"]),
    ("auto_7b_eps_bad", ["autoscale", *scen("7b", "64"), "--synth", BURST, "--mode", "operator",
                         "--epsilon", "0.05", "--slo-prefill", "0.4", "--slo-decode", "0.04"]),
    ("auto_70b_operator", ["autoscale", *scen("70b", "1k"), "--synth",
                           "burst:rate=8,duration=300,period=600,burst_factor=4,input_sigma=0.8,output_sigma=0.6",
                           "--mode", "operator", "--slo-prefill", "2.0", "--slo-decode", "0.15"]),
    ("auto_70b_model_default", ["autoscale", *scen("70b", "1k"), "--synth",
                                "burst:rate=8,duration=300,period=600,burst_factor=4,input_sigma=0.8",
                                "--mode", "model", "--placement", "default_stream",
                                "--slo-prefill", "2.0", "--slo-decode", "0.15"]),
    ("auto_mm_hetero", ["autoscale", *scen("mm", "hetero"), "--synth",
                        "diurnal:rate=6,duration=300,period=300,amplitude=0.5,input_median=768,input_sigma=1.5",
                        "--mode", "operator", "--slo-prefill", "1.0", "--slo-decode", "0.08", "--seed", "1"]),
    ("auto_trace_gap", ["autoscale", *scen("7b", "64"), "--trace", "trace_gap.csv", "--mode", "operator"]),
    ("auto_trace_gap_quantile", ["autoscale", *scen("7b", "64"), "--trace", "trace_gap.csv", "--mode", "model",
                                 "--window-len", "45", "--quantile", "0.5"]),
    ("auto_tiny_oracle", ["autoscale", *scen("tiny", "64"), "--synth", "constant:rate=20,duration=120,seqlen=1024",
                          "--mode", "oracle"]),
    ("auto_7b_oracle_guard", ["autoscale", *scen("7b", "64"), "--synth", "constant:rate=5,duration=60",
                              "--mode", "oracle"]),
    ("auto_7b_infeasible", ["autoscale", *scen("7b", "64"), "--synth", BURST, "--mode", "operator",
                            "--slo-prefill", "0.02", "--slo-decode", "0.002"]),
    ("auto_fleet_exhausted", ["autoscale", *scen("7b", "4"), "--synth",
                              "diurnal:rate=8,amplitude=0.9,period=600,duration=600,seqlen=4096",
                              "--mode", "operator"]),
    ("auto_bad_slo", ["autoscale", *scen("7b", "64"), "--synth", BURST, "--slo-decode", "-1"]),
    ("sweep_seqlen", ["sweep", *scen("7b", "64"), "--synth", "constant:rate=30,seqlen=4096", "--sweep", "seqlen",
                      "--range", "1024,2048,4096,8192,16384"]),
    ("sweep_seqlen_default", ["sweep", *scen("7b", "64"), "--synth", "constant:rate=30,seqlen=4096",
                              "--sweep", "seqlen", "--range", "1024,4096,8192", "--placement", "default_stream"]),
    ("sweep_qps", ["sweep", *scen("7b", "64"), "--synth", "constant:rate=30,seqlen=2048", "--sweep", "qps",
                   "--range", "0,1,5,10,15,40,80"]),
    ("sweep_model_scale", ["sweep", *scen("70b", "1k"), "--synth", "constant:rate=20,seqlen=1024",
                           "--sweep", "model_scale", "--range", "0.5,1,1.5", "--slo-prefill", "2.0"]),
    ("sweep_mm_qps_hetero", ["sweep", *scen("mm", "hetero"), "--synth", "constant:rate=10,seqlen=768",
                             "--sweep", "qps", "--range", "2,10,30", "--slo-prefill", "1.0"]),
    ("sweep_infeasible", ["sweep", *scen("7b", "64"), "--synth", "constant:rate=30,seqlen=4096", "--sweep", "qps",
                          "--range", "10,30", "--slo-prefill", "0.01"]),
]


def run_case(argv, run_main):
    """Run a CLI main() from tests/golden/cli/ into a scratch --out; returns
    (exit code, stderr, {file: bytes})."""
    with tempfile.TemporaryDirectory() as tmp:
        out = os.path.join(tmp, "out")
        err = io.StringIO()
        cwd = os.getcwd()
        os.chdir(IN)
        try:
            with contextlib.redirect_stderr(err):
                rc = run_main(argv + ["--out", out])
        finally:
            os.chdir(cwd)
        files = {}
        if os.path.isdir(out):
            for name in sorted(os.listdir(out)):
                with open(os.path.join(out, name), "rb") as fh:
                    files[name] = fh.read()
        return rc, err.getvalue(), files


def summarize(rc, err, files):
    return {"exit": rc, "stderr": err,
            "files": {k: hashlib.sha256(v).hexdigest() for k, v in files.items()},
            "texts": {k: v.decode() for k, v in files.items() if k.endswith(".csv")}}


def main():
    write_inputs()
    out = []
    for name, argv in CASES:
        rc, err, files = run_case(argv, ref_cli.main)
        rec = {"name": name, "argv": argv, **summarize(rc, err, files)}
        out.append(rec)
        print(f"{name}: exit {rc}, {len(files)} files {err.strip()[:80]}")
    with open(os.path.join(HERE, "cli.json"), "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
