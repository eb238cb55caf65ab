export PYTHONPATH=$PWD
timeout 2400 compute-sanitizer --tool racecheck --kernel-name kns=greedy --error-exitcode 9 python -m pytest -x -q tests/test_gpu_parity.py -k "golden_greedy or full_trace_greedy" > gpurun_out/rc_greedy.log 2>&1
echo "racecheck greedy rc=$? $(grep -E 'passed|failed' gpurun_out/rc_greedy.log | tail -1) $(grep -E 'SUMMARY' gpurun_out/rc_greedy.log | tail -1)"
timeout 2400 compute-sanitizer --tool synccheck --kernel-name kns=greedy --error-exitcode 9 python -m pytest -x -q tests/test_gpu_parity.py -k "golden_greedy" > gpurun_out/sc_greedy.log 2>&1
echo "synccheck greedy rc=$? $(grep -E 'passed|failed' gpurun_out/sc_greedy.log | tail -1) $(grep -E 'SUMMARY' gpurun_out/sc_greedy.log | tail -1)"
timeout 1200 compute-sanitizer --tool memcheck --kernel-name kns=greedy --error-exitcode 9 python -m pytest -x -q tests/test_gpu_parity.py -k "golden_greedy" > gpurun_out/mc_greedy.log 2>&1
echo "memcheck greedy rc=$? $(grep -E 'passed|failed' gpurun_out/mc_greedy.log | tail -1) $(grep -E 'SUMMARY' gpurun_out/mc_greedy.log | tail -1)"
