# same-box A/B of prebuilt libraries tools/ab/lib<V>.so (V in $VARIANTS, default "A B"):
# runs $CMD (default: quick_time over $CFGS) per variant, interleaved, 3 reps -> gpurun_out/ab.txt
export PYTHONPATH=$PWD
for rep in 1 2 3; do
  for v in ${VARIANTS:-A B}; do
    if [ -n "$CMD" ]; then
      echo "$v $(OPSC_LIB_PATH=$PWD/tools/ab/lib$v.so bash -c "$CMD" 2>&1 | tail -1)"
    else
      for c in ${CFGS:-cfg2 cfg3 cfg5}; do
        echo "$v $(OPSC_LIB_PATH=$PWD/tools/ab/lib$v.so python tools/quick_time.py $c 2>&1 | head -1)"
      done
    fi
  done
done > gpurun_out/ab.txt
