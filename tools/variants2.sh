#!/bin/bash
# Build compose-kernel variants on the GPU box and time cfg5 + cfg2 (dev tool).
export PYTHONPATH=$PWD
for v in "$@"; do
  OPSC_NVCC_EXTRA="$v" python -m paper_2511_02248_b200.build --force > /dev/null 2>&1 || { echo "build failed $v"; continue; }
  echo "variant [$v]: $(python tools/quick_time.py cfg5 2>/dev/null | head -1) | $(python tools/quick_time.py cfg2 2>/dev/null | head -1)"
done
python -m paper_2511_02248_b200.build --force > /dev/null 2>&1
