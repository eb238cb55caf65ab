# pow / placement iteration: GPU suite, fuzz at 3000 cases, placement timing (arg 1 = tag)
export PYTHONPATH=$PWD
tag=${1:-pw}
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/${tag}_tests.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_tests.log
OPSC_FUZZ_CASES=3000 timeout 900 python -m pytest tests/test_gpu_fuzz_reference.py -q -p no:cacheprovider > gpurun_out/${tag}_big.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_big.log
timeout 300 python bench.py --steps 3 --warmup 3 > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
