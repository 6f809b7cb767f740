#!/bin/bash
# ncu --set full of the K3b kernel at a BASELINE config: tools/k3_ncu.sh <config>
C=$1; O=gpurun_out/k3n; mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k3b' -c 1 -o $O/k3b_cfg$C -f python tools/k3_sweep.py $C - > $O/ncu_$C.log 2>&1; echo ncu rc=$?
