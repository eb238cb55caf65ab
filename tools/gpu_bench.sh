# full bench line (both arms) + launch list of the bench command (arg 1 = tag)
export PYTHONPATH=$PWD
tag=${1:-bench}
timeout 900 python bench.py > gpurun_out/${tag}.json 2> gpurun_out/${tag}.err
timeout 900 python bench.py --impl reference > gpurun_out/${tag}_ref.json 2> gpurun_out/${tag}_ref.err
if [ -n "$2" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${tag}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-latency > /dev/null 2>&1
fi
