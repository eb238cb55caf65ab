# W=1 per-window pipeline: tests, latency per mode, fine-sampled ncu of materialize and greedy phase 1 (decode window) (arg 1 = tag)
export PYTHONPATH=$PWD
tag=${1:-w1}
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/${tag}_tests.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_tests.log
for m in operator model oracle; do timeout 300 python tools/w1_latency.py $m 60; done > gpurun_out/${tag}_w1.txt 2>&1
timeout 600 ncu --set full --import-source on --clock-control none --warp-sampling-interval 0 -k regex:materialize -s 3 -c 1 -o gpurun_out/${tag}_mat -f python tools/w1_profile.py model 7 prefill > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none --warp-sampling-interval 0 -k regex:greedy -s 4 -c 1 -o gpurun_out/${tag}_gdec -f python tools/w1_profile.py operator 7 decode > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_ops_prefill.csv python tools/w1_profile.py operator 7 prefill > /dev/null 2>&1
