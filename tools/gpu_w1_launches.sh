export PYTHONPATH=$PWD
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/w1ops_decode.csv python tools/w1_profile.py operator 7 decode > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/w1ops_prefill.csv python tools/w1_profile.py operator 7 prefill > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/w1model.csv python tools/w1_profile.py model 7 prefill > /dev/null 2>&1
