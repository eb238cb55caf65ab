export PYTHONPATH=$PWD
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02_gpu.txt
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02_gputests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r02_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/r02_bench_ref.json 2> gpurun_out/r02_bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-latency > gpurun_out/r02_ncu_bench.log 2>&1
timeout 300 python tools/api_latency.py > gpurun_out/r02_api_latency.txt 2>&1
ls -la gpurun_out
