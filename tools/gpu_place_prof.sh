# placement kernel: full ncu capture with source-level warp sampling (trace pipeline, cfg2 70B, 60 windows)
export PYTHONPATH=$PWD
timeout 600 ncu --set full --import-source on --clock-control none --warp-sampling-interval 0 -k regex:place_kernel -c 1 \
  -o gpurun_out/${1:-place} -f python tools/profile_pipeline.py operator > gpurun_out/${1:-place}.log 2>&1
