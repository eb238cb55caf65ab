#!/bin/bash
# compute-sanitizer (memcheck / racecheck / synccheck / initcheck) over the
# library's kernels on the GPU box: the smoke entry (all three planner modes +
# shared placement) and the compose / windowize / pipeline GPU tests at
# small sizes. Logs land in gpurun_out/sanitize_<tool>.log.
export PYTHONPATH=$PWD
mkdir -p gpurun_out
SMOKE='import __graft_entry__ as g; g.smoke()'
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $tool --kernel-name kns=opsc --error-exitcode 9 \
    python -c "$SMOKE" > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool smoke rc=$?"
done
timeout 1500 compute-sanitizer --tool memcheck --kernel-name kns=opsc --error-exitcode 9 \
  python -m pytest -x -q tests/test_gpu_compose_edges.py tests/test_gpu_windowize.py tests/test_gpu_place.py \
  -k "not flat" > gpurun_out/sanitize_memcheck_tests.log 2>&1
echo "memcheck tests rc=$?"
timeout 1500 compute-sanitizer --tool racecheck --kernel-name kns=opsc --error-exitcode 9 \
  python -m pytest -x -q tests/test_gpu_compose_edges.py tests/test_gpu_windowize.py -k "not flat" \
  > gpurun_out/sanitize_racecheck_tests.log 2>&1
echo "racecheck tests rc=$?"
