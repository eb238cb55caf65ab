#!/bin/bash
# K2 variants (dev tool, GPU box): unroll of the last middle level's loop.
export PYTHONPATH=$PWD
for u in 1 2 3; do
  OPSC_NVCC_EXTRA="-DOPSC_COMPOSE_LUNROLL=$u" python -m paper_2511_02248_b200.build --force > /dev/null 2>&1 || echo "build fail $u"
  for c in cfg5 cfg2 cfg3; do echo "lunroll=$u $(python tools/quick_time.py $c 2>&1 | grep rate)"; done
done
python -m paper_2511_02248_b200.build --force > /dev/null 2>&1
