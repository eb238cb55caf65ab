# round-end style run: full GPU suite, smoke, both bench arms, launch list, API latency, W=1 latency (arg 1 = tag)
export PYTHONPATH=$PWD
tag=${1:-final}
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/${tag}_tests.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_smoke.log
timeout 900 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/${tag}_bench_ref.json 2> gpurun_out/${tag}_bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${tag}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-latency > /dev/null 2>&1
timeout 300 python tools/api_latency.py 60 > gpurun_out/${tag}_api.txt 2>&1
timeout 300 python tools/api_breakdown.py >> gpurun_out/${tag}_api.txt 2>&1
for m in operator model oracle; do timeout 300 python tools/w1_latency.py $m 60; done > gpurun_out/${tag}_w1.txt 2>&1
