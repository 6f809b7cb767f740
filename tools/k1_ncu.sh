#!/bin/bash
# ncu --set full of the stage-1 kernel at a BASELINE config: tools/k1_ncu.sh <config> <tag>
C=$1; T=${2:-k1}
O=gpurun_out/$T; mkdir -p $O
python tools/k1_sweep.py $C - 2>&1 | tail -1 | tee $O/time_config$C.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k1s_kernel|k1t_kernel|k1v2|k1_csr' -c 1 -o $O/k1_cfg$C -f python tools/k1_sweep.py $C - > $O/ncu_$C.log 2>&1; echo ncu rc=$?
