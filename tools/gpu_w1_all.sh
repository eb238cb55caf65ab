# full GPU suite + W=1 latency for every mode + per-point API (arg 1 = tag)
export PYTHONPATH=$PWD
tag=${1:-w1}
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/${tag}_tests.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_tests.log
for m in operator model oracle; do timeout 300 python tools/w1_latency.py $m 60; done > gpurun_out/${tag}_w1.txt 2>&1
timeout 300 python tools/api_latency.py 60 > gpurun_out/${tag}_api.txt 2>&1
