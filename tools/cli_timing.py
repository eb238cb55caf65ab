"""Wall time of `autoscale` over the 1-hour 70B trace (60 windows x 2 phases,
plan + place + all artifacts written) through this package's CLI.

    python tools/cli_timing.py [--reference]   # --reference: the reference CLI (build container)

Writes gpurun_out/cli_timing.json.
"""

import json
import os
import sys
import tempfile
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
IN = os.path.join(REPO, "tests", "golden", "cli")

ARGS = ["autoscale", "--dag", "dag_70b.json", "--profiles", "profiles_70b.json", "--fleet", "fleet_1k.json",
        "--synth", "burst:rate=8,duration=3600,period=600,burst_factor=4,input_sigma=0.8,output_sigma=0.6",
        "--slo-prefill", "2.0", "--slo-decode", "0.15"]


def main():
    if "--reference" in sys.argv:
        sys.path.insert(0, "/root/reference/pkg/src")
        from opscaler import cli
        reps = 1
    else:
        from paper_2511_02248_b200 import cli
        reps = 5
    os.chdir(IN)
    res = {}
    for mode in ("operator", "model"):
        for placement in ("shared", "default_stream"):
            times = []
            for r in range(reps + (0 if reps == 1 else 1)):
                with tempfile.TemporaryDirectory() as tmp:
                    t = time.perf_counter()
                    rc = cli.main(ARGS + ["--mode", mode, "--placement", placement, "--out", tmp])
                    times.append(time.perf_counter() - t)
                    assert rc == 0
            times = times if reps == 1 else times[1:]  # first run: CUDA context + library load
            res[f"{mode}/{placement}"] = {"median_s": sorted(times)[len(times) // 2], "runs": times}
            print(mode, placement, res[f"{mode}/{placement}"]["median_s"], flush=True)
    os.makedirs(os.path.join(REPO, "gpurun_out"), exist_ok=True)
    name = "cli_timing_reference.json" if "--reference" in sys.argv else "cli_timing.json"
    with open(os.path.join(REPO, "gpurun_out", name), "w") as fh:
        json.dump(res, fh, indent=1)


if __name__ == "__main__":
    main()
