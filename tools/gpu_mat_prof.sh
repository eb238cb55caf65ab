export PYTHONPATH=$PWD
timeout 600 ncu --set full --import-source on --clock-control none --warp-sampling-interval 0 -k regex:materialize -s 2 -c 1 -o gpurun_out/mat_w1 -f python tools/w1_profile.py model 7 prefill > gpurun_out/mat_w1.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none --warp-sampling-interval 0 -k regex:materialize -s 2 -c 1 -o gpurun_out/mat_w1_oracle -f python tools/w1_profile.py oracle 7 prefill > gpurun_out/mat_w1o.log 2>&1
