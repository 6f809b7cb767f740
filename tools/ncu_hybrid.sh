#!/bin/bash
# Can ncu profile the hybrid LU when it is launched without the cooperative attribute?
O=gpurun_out/hyb; mkdir -p $O
SRLU_LU_NOCOOP=1 python tools/lu_time.py 16384 110 | tee $O/nocoop_time.txt
python tools/lu_time.py 16384 110 | tee -a $O/nocoop_time.txt
env | grep -i "inject\|nsight" > $O/env_outside.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lu_hybrid -c 1 -o $O/lu_hybrid_cfg2 -f python tools/run_lu_once.py > $O/ncu.log 2>&1; echo "ncu rc=$?" | tee -a $O/ncu.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_config2.csv python tools/one_decomp.py 2 1 > $O/ncu_launches.log 2>&1; echo "ncu launches rc=$?" | tee -a $O/ncu.log
python tools/launch_table.py $O/launches_config2.csv | tail -40
