#!/bin/bash
# K2 variants (dev tool, GPU box): unroll of the shared-memory k loop (12..32-entry tiles).
export PYTHONPATH=$PWD
for u in ${KU_LIST:-1 2 3 4 6}; do
  OPSC_NVCC_EXTRA="-DOPSC_COMPOSE_KUNROLL=$u" python -m paper_2511_02248_b200.build --force > /dev/null 2>&1 || echo "build fail $u"
  r=$(grep -A2 "compose_kernelILi24ELi2ELb0" paper_2511_02248_b200/_lib/ptxas.log | grep -o "[0-9]* bytes spill stores\|Used [0-9]* registers" | tr '\n' ' ')
  for c in cfg5 cfg1; do echo "kunroll=$u [$r] $(python tools/quick_time.py $c 2>&1 | grep rate)"; done
done
python -m paper_2511_02248_b200.build --force > /dev/null 2>&1
