#!/bin/bash
# ncu --set full of ONE cfg5 compose launch per build variant (dev tool, GPU box).
# usage: tools/ncu_compose.sh tag1 "<nvcc flags 1>" tag2 "<nvcc flags 2>" ...
export PYTHONPATH=$PWD
mkdir -p gpurun_out
while [ $# -ge 2 ]; do
  tag=$1; flags=$2; shift 2
  OPSC_NVCC_EXTRA="$flags" python -m paper_2511_02248_b200.build --force > /dev/null 2>&1 || { echo "build failed $tag"; continue; }
  echo "variant $tag [$flags]: $(python tools/quick_time.py 2>&1 | head -1)"
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:compose_kernel -s 3 -c 1 \
    -o gpurun_out/compose_$tag -f python tools/quick_time.py > gpurun_out/ncu_$tag.log 2>&1
  echo "ncu $tag rc=$?"
done
python -m paper_2511_02248_b200.build --force > /dev/null 2>&1
