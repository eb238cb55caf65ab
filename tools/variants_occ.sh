#!/bin/bash
# K2 occupancy variants (dev tool, GPU box): CTA size x min CTAs per SM.
export PYTHONPATH=$PWD
for v in "256 3" "128 7" "192 5" "128 6" "64 14"; do
  set -- $v
  OPSC_NVCC_EXTRA="-DOPSC_COMPOSE_THREADS=$1 -DOPSC_COMPOSE_MINB=$2" python -m paper_2511_02248_b200.build --force > /dev/null 2>&1 || echo "build fail $v"
  r=$(grep -A2 "compose_kernelILi24ELi2ELb0" paper_2511_02248_b200/_lib/ptxas.log | grep -o "[0-9]* bytes spill stores\|Used [0-9]* registers" | tr '\n' ' ')
  for c in cfg5 cfg2; do echo "occ=$1x$2 [$r] $(python tools/quick_time.py $c 2>&1 | grep rate)"; done
done
python -m paper_2511_02248_b200.build --force > /dev/null 2>&1
