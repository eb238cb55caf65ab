#!/bin/bash
# Build compose-kernel variants on the GPU box and time cfg5 (dev tool).
export PYTHONPATH=$PWD
for v in "" "-DOPSC_COMPOSE_MINB=4" "-DOPSC_COMPOSE_MINB=2" "-DOPSC_COMPOSE_THREADS=512 -DOPSC_COMPOSE_MINB=1"; do
  OPSC_NVCC_EXTRA="$v" python -m paper_2511_02248_b200.build --force > /dev/null 2>&1 || { echo "build failed $v"; continue; }
  echo "variant [$v]: $(python tools/quick_time.py 2>&1 | head -1)"
done
python -m paper_2511_02248_b200.build --force > /dev/null 2>&1
