#!/bin/bash
# Build greedy-kernel variants on the GPU box and time W=1 / batched greedy (dev tool).
export PYTHONPATH=$PWD
for v in "$@"; do
  OPSC_NVCC_EXTRA="$v" python -m paper_2511_02248_b200.build --force > /dev/null 2>&1 || { echo "build failed $v"; continue; }
  echo "variant [$v]: $(python tools/w1_latency.py operator 60 2>/dev/null | tail -1)"
done
python -m paper_2511_02248_b200.build --force > /dev/null 2>&1
