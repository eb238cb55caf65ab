export PYTHONPATH=$PWD
timeout 600 python -m pytest tests/test_gpu_certify.py tests/test_abi.py -x -q -p no:cacheprovider > gpurun_out/r02_cert_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02_cert_tests.log
timeout 600 python bench.py --no-cpu-baseline --no-latency > gpurun_out/r02_cert_bench.json 2> gpurun_out/r02_cert_bench.err
