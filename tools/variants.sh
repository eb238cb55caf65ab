#!/bin/bash
# Build compose-kernel variants on the GPU box and time cfg5 (dev tool).
# usage: tools/variants.sh "<nvcc flags variant 1>" "<variant 2>" ...
export PYTHONPATH=$PWD
for v in "$@"; do
  OPSC_NVCC_EXTRA="$v" python -m paper_2511_02248_b200.build --force > /dev/null 2>&1 || { echo "build failed $v"; continue; }
  echo "variant [$v]: $(python tools/quick_time.py 2>&1 | head -1)"
done
python -m paper_2511_02248_b200.build --force > /dev/null 2>&1
