#!/bin/bash
# K2 variants (dev tool, GPU box): min CTAs per SM for the small register tiles (NJ <= 8).
export PYTHONPATH=$PWD
for m in ${MINB_LIST:-3 4 5}; do
  OPSC_NVCC_EXTRA="-DOPSC_COMPOSE_MINB_SMALL=$m" python -m paper_2511_02248_b200.build --force > /dev/null 2>&1 || echo "build fail $m"
  r=$(grep -A2 "compose_kernelILi6ELi2ELb1" paper_2511_02248_b200/_lib/ptxas.log | grep -o "[0-9]* bytes spill stores\|Used [0-9]* registers" | tr '\n' ' ')
  for c in cfg2 cfg3; do echo "minb_small=$m [$r] $(python tools/quick_time.py $c 2>&1 | grep rate)"; done
done
python -m paper_2511_02248_b200.build --force > /dev/null 2>&1
