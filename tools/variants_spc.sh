#!/bin/bash
# K2 variants (dev tool, GPU box): slices per CTA (OPSC_COMPOSE_SPC override).
export PYTHONPATH=$PWD
for s in 1 2 4 8 16 32 auto; do
  if [ $s = auto ]; then unset OPSC_COMPOSE_SPC; else export OPSC_COMPOSE_SPC=$s; fi
  for c in cfg5 cfg2 cfg3; do echo "spc=$s $(python tools/quick_time.py $c 2>&1 | grep rate)"; done
done
