set -x
export PYTHONPATH=$PWD
timeout 600 ncu --set full --import-source on --clock-control none -k regex:compose_kernel -s 3 -c 1 -o gpurun_out/r02_k2_cfg2 -f python tools/quick_time.py cfg2 > gpurun_out/r02_ncu_k2_cfg2.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:greedy -s 4 -c 2 -o gpurun_out/r02_greedy_w1 -f python tools/w1_profile.py operator 7 prefill > gpurun_out/r02_ncu_greedy.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:place -c 1 -o gpurun_out/r02_place -f python tools/profile_pipeline.py operator > gpurun_out/r02_ncu_place.log 2>&1
python tools/quick_time.py cfg2 > gpurun_out/r02_qt_cfg2.txt 2>&1
python tools/quick_time.py cfg5 > gpurun_out/r02_qt_cfg5.txt 2>&1
python tools/w1_latency.py > gpurun_out/r02_w1_latency.txt 2>&1
ls -la gpurun_out
