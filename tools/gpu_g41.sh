export PYTHONPATH=$PWD
timeout 600 ncu --set full --import-source on --clock-control none --warp-sampling-interval 0 -k regex:greedy -s 4 -c 2 -o gpurun_out/g${W:-41} -f python tools/w1_profile.py operator ${W:-41} prefill > gpurun_out/g${W:-41}.log 2>&1
