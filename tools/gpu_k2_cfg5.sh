export PYTHONPATH=$PWD
timeout 900 ncu --set full --import-source on --clock-control none --warp-sampling-interval 4 -k regex:compose_kernel -s 3 -c 1 -o gpurun_out/k2_cfg5 -f python tools/quick_time.py cfg5 > gpurun_out/k2_cfg5.log 2>&1
