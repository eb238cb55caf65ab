export PYTHONPATH=$PWD
SMOKE='import __graft_entry__ as g; g.smoke()'
timeout 1200 compute-sanitizer --tool synccheck --kernel-name kns=opsc --error-exitcode 9 python -c "$SMOKE" > gpurun_out/sanitize_synccheck.log 2>&1
echo "synccheck smoke rc=$? $(grep -E 'SUMMARY' gpurun_out/sanitize_synccheck.log | tail -1)"
timeout 1200 compute-sanitizer --tool synccheck --kernel-name kns=opsc --error-exitcode 9 python -m pytest -x -q tests/test_gpu_fused.py tests/test_gpu_certify.py tests/test_gpu_place.py > gpurun_out/sanitize_synccheck_tests.log 2>&1
echo "synccheck tests rc=$? $(grep -E 'passed|failed' gpurun_out/sanitize_synccheck_tests.log | tail -1) $(grep -E 'SUMMARY' gpurun_out/sanitize_synccheck_tests.log | tail -1)"
timeout 600 python -m pytest -x -q tests/test_gpu_fused.py tests/test_gpu_parity.py > gpurun_out/sync_fix_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/sync_fix_tests.log
