export PYTHONPATH=$PWD
for rep in 1 2; do for spc in 1 2 4 8; do echo "spc=$spc $(OPSC_COMPOSE_SPC=$spc python tools/quick_time.py cfg5 | head -1)"; done; done > gpurun_out/spc.txt
for rep in 1 2; do for spc in 1 2 4; do echo "cfg2 spc=$spc $(OPSC_COMPOSE_SPC=$spc python tools/quick_time.py cfg2 | head -1)"; done; done >> gpurun_out/spc.txt
