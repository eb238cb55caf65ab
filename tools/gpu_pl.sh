export PYTHONPATH=$PWD
timeout 900 python -m pytest tests/test_gpu_place.py tests/test_gpu_pipeline.py tests/test_gpu_cli.py tests/test_gpu_dropin.py -x -q -p no:cacheprovider > gpurun_out/pl_tests.log 2>&1; echo "rc=$?" >> gpurun_out/pl_tests.log
timeout 300 ncu --metrics gpu__time_duration.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none --csv -k regex:place --log-file gpurun_out/pl_pipe.csv python tools/profile_pipeline.py operator > /dev/null 2>&1
