# API latency iteration: drop-in + planner GPU tests, per-point latency and its breakdown (arg 1 = tag)
export PYTHONPATH=$PWD
tag=${1:-api}
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/${tag}_tests.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_tests.log
for i in 1 2; do timeout 300 python tools/api_latency.py 60; done > gpurun_out/${tag}_api.txt 2>&1
timeout 300 python tools/api_breakdown.py >> gpurun_out/${tag}_api.txt 2>&1
