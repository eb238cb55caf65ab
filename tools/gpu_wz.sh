export PYTHONPATH=$PWD
timeout 900 python -m pytest tests/test_gpu_windowize.py tests/test_gpu_pipeline.py tests/test_gpu_cli.py -x -q -p no:cacheprovider > gpurun_out/wz_tests.log 2>&1; echo "rc=$?" >> gpurun_out/wz_tests.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/wz_pipe.csv python tools/profile_pipeline.py operator > /dev/null 2>&1
timeout 600 python bench.py --no-cpu-baseline --steps 3 --warmup 3 > gpurun_out/wz_bench.json 2>/dev/null
