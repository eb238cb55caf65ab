# greedy W=1 source-level capture of both phases + the W=1 operator pipeline's launch list (arg 1 = tag)
export PYTHONPATH=$PWD
tag=${1:-gs}
timeout 600 ncu --set full --import-source on --clock-control none -k regex:greedy -s 4 -c 2 -o gpurun_out/${tag}_greedy -f python tools/w1_profile.py operator 7 prefill > gpurun_out/${tag}_ncu_greedy.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/${tag}_w1_launches.csv python tools/w1_profile.py operator 7 prefill > gpurun_out/${tag}_w1l.log 2>&1
