export PYTHONPATH=$PWD
timeout 600 python -m pytest tests/test_gpu_certify.py -x -q -p no:cacheprovider > gpurun_out/r02_cert_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02_cert_tests.log
bash tools/ncu_r02a.sh
