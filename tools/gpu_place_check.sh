# placement kernel: GPU tests, then compute-sanitizer (memcheck / racecheck / synccheck / initcheck) on them
export PYTHONPATH=$PWD
timeout 900 python -m pytest tests/test_gpu_place.py -x -q -p no:cacheprovider > gpurun_out/plc_tests.log 2>&1; echo "rc=$?" >> gpurun_out/plc_tests.log
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --kernel-name kns=place_kernel --error-exitcode 9 \
    python -m pytest -x -q -p no:cacheprovider tests/test_gpu_place.py -k "large_plans or probe_chunk or odd" > gpurun_out/plc_san_$tool.log 2>&1
  echo "$tool rc=$? $(grep -E 'passed|failed' gpurun_out/plc_san_$tool.log | tail -1) $(grep -E 'SUMMARY' gpurun_out/plc_san_$tool.log | tail -1)" >> gpurun_out/plc_tests.log
done
