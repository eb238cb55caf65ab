# K2 A/B on one box: quick_time for cfg2 / cfg3 / cfg5, compose edge + parity tests,
# optional ncu --set full of the cfg2 compose launch (arg 1 = tag)
export PYTHONPATH=$PWD
tag=${1:-k2}
for c in cfg2 cfg3 cfg5; do python tools/quick_time.py $c 2>&1 | head -1; done > gpurun_out/${tag}_qt.txt
timeout 900 python -m pytest tests/test_gpu_compose_edges.py tests/test_gpu_parity.py tests/test_gpu_certify.py -x -q -p no:cacheprovider > gpurun_out/${tag}_tests.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_tests.log
if [ -n "$2" ]; then
timeout 600 ncu --set full --import-source on --clock-control none --warp-sampling-interval 0 -k regex:compose_kernel -s 3 -c 1 -o gpurun_out/${tag}_cfg2 -f python tools/quick_time.py cfg2 > gpurun_out/${tag}_ncu.log 2>&1
fi
