# same-box A/B of two prebuilt libraries (tools/ab/libA.so, libB.so): quick_time per config, interleaved
export PYTHONPATH=$PWD
for rep in 1 2 3; do
  for v in A B; do
    for c in ${CFGS:-cfg2 cfg3 cfg5}; do
      echo "$v $(OPSC_LIB_PATH=$PWD/tools/ab/lib$v.so python tools/quick_time.py $c 2>&1 | head -1)"
    done
  done
done > gpurun_out/ab.txt
