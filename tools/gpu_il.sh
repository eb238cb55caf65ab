export PYTHONPATH=$PWD
for c in cfg2 cfg3; do for il in 3 4 5 6; do echo "$c IL=$il $(OPSC_COMPOSE_IL=$il python tools/quick_time.py $c | head -1)"; done; done > gpurun_out/il.txt 2>&1
for c in cfg2 cfg3; do echo "$c auto $(python tools/quick_time.py $c | head -1)"; done >> gpurun_out/il.txt
