"""Generate per-window trace statistics with the REFERENCE implementation.

Runs only in the build container (it imports the read-only reference from
/root/reference). Writes workloads/traces.npz: for every
config in scenarios.TRACES, the reference's synth_workload(spec, seed)
(workload.py:195-232) cut by windowize (workload.py:114-158) into
prefill/decode demand points.

    PYTHONHASHSEED=0 python tests/golden/make_traces.py
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, "/root/reference/pkg/src")

from opscaler import workload as ref_wl  # noqa: E402

from paper_2511_02248_b200.scenarios import TRACES  # noqa: E402


def main():
    out = {}
    for name, cfg in TRACES.items():
        recs = ref_wl.synth_workload(ref_wl.SynthSpec(**cfg["spec"]), seed=cfg["seed"])
        wins = ref_wl.windowize(recs, window_len=cfg["window_len"], quantile=cfg["quantile"])
        out[f"{name}/prefill_qps"] = np.array([p.qps for p, _ in wins], dtype=np.float64)
        out[f"{name}/prefill_len"] = np.array([p.seq_len for p, _ in wins], dtype=np.int32)
        out[f"{name}/decode_qps"] = np.array([d.qps for _, d in wins], dtype=np.float64)
        out[f"{name}/decode_len"] = np.array([d.seq_len for _, d in wins], dtype=np.int32)
        out[f"{name}/t0"] = np.array([p.window[0] for p, _ in wins], dtype=np.float64)
        out[f"{name}/t1"] = np.array([p.window[1] for p, _ in wins], dtype=np.float64)
        out[f"{name}/n_records"] = np.array([len(recs)], dtype=np.int64)
        # checksum of the raw record stream, to pin the workload.py mirror
        arr = np.array([(r.arrival_time, r.input_len, r.output_len) for r in recs[:5000]],
                       dtype=np.float64)
        out[f"{name}/head_records"] = arr
        print(name, len(recs), "records", len(wins), "windows")
    path = os.path.join(REPO, "workloads", "traces.npz")
    np.savez_compressed(path, **out)
    print("wrote", path)


if __name__ == "__main__":
    main()
