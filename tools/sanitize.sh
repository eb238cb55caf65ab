#!/bin/bash
# compute-sanitizer (memcheck / racecheck / synccheck / initcheck) over the
# library's kernels on the GPU box: the smoke entry (all three planner modes +
# shared placement) and GPU tests at small sizes. Logs land in
# gpurun_out/sanitize_<tool>*.log; a summary line per run on stdout.
export PYTHONPATH=$PWD
mkdir -p gpurun_out
SMOKE='import __graft_entry__ as g; g.smoke()'
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $tool --kernel-name kns=opsc --error-exitcode 9 \
    python -c "$SMOKE" > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool smoke rc=$? $(grep -E 'SUMMARY' gpurun_out/sanitize_$tool.log | tail -1)"
done
TESTS="tests/test_gpu_compose_edges.py tests/test_gpu_windowize.py tests/test_gpu_place.py tests/test_gpu_model_table.py tests/test_gpu_certify.py tests/test_gpu_fused.py"
for tool in memcheck racecheck; do
  timeout 2400 compute-sanitizer --tool $tool --kernel-name kns=opsc --error-exitcode 9 \
    python -m pytest -x -q $TESTS -k "not flat and not level_splits" > gpurun_out/sanitize_${tool}_tests.log 2>&1
  echo "$tool tests rc=$? $(grep -E 'passed|failed' gpurun_out/sanitize_${tool}_tests.log | tail -1) $(grep -E 'SUMMARY' gpurun_out/sanitize_${tool}_tests.log | tail -1)"
done
timeout 2400 compute-sanitizer --tool memcheck --kernel-name kns=opsc --error-exitcode 9 \
  python -m pytest -x -q tests/test_gpu_parity.py -k "golden_greedy or golden_model or golden_oracle" > gpurun_out/sanitize_memcheck_golden.log 2>&1
echo "memcheck golden rc=$? $(grep -E 'passed|failed' gpurun_out/sanitize_memcheck_golden.log | tail -1)"
timeout 2400 compute-sanitizer --tool racecheck --kernel-name kns=opsc --error-exitcode 9 \
  python -m pytest -x -q tests/test_gpu_parity.py -k "golden_greedy" > gpurun_out/sanitize_racecheck_greedy.log 2>&1
echo "racecheck greedy goldens rc=$? $(grep -E 'passed|failed' gpurun_out/sanitize_racecheck_greedy.log | tail -1) $(grep -E 'SUMMARY' gpurun_out/sanitize_racecheck_greedy.log | tail -1)"
