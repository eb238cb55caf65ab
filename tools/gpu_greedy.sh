# greedy / placement iteration: full GPU suite, W=1 latency, fine-sampled ncu of greedy W=1 and of place (arg 1 = tag)
export PYTHONPATH=$PWD
tag=${1:-gr}
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/${tag}_tests.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_tests.log
timeout 300 python tools/w1_latency.py operator 60 > gpurun_out/${tag}_w1.txt 2>&1
timeout 600 ncu --set full --import-source on --clock-control none --warp-sampling-interval 0 -k regex:greedy -s 4 -c 2 -o gpurun_out/${tag}_greedy -f python tools/w1_profile.py operator 7 prefill > gpurun_out/${tag}_ncu_greedy.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none --warp-sampling-interval 2 -k regex:place -c 1 -o gpurun_out/${tag}_place -f python tools/profile_pipeline.py operator > gpurun_out/${tag}_ncu_place.log 2>&1
timeout 300 python tools/api_latency.py 60 > gpurun_out/${tag}_api.txt 2>&1
timeout 300 python tools/api_breakdown.py >> gpurun_out/${tag}_api.txt 2>&1
