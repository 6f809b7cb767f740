#!/bin/bash
# K1T timing under debug knobs + one ncu --set full capture of k1t_kernel (config 2 shape)
O=gpurun_out/k1t; mkdir -p $O
for d in 0 1 2 3 4 7; do SRLU_K1T_DBG=$d python tools/k1_sweep.py 2 - 2>&1 | tail -1 | sed "s/^/dbg=$d /"; done | tee $O/dbg_sweep.txt
for ns in 3 4 5; do SRLU_K1T_NS=$ns python tools/k1_sweep.py 2 - 2>&1 | tail -1 | sed "s/^/ns=$ns /"; done | tee -a $O/dbg_sweep.txt
for r in 32 28 24 16; do SRLU_K1T_ROWS=$r python tools/k1_sweep.py 2 - 2>&1 | tail -1 | sed "s/^/rows=$r /"; done | tee -a $O/dbg_sweep.txt
python tools/k1_sweep.py 2 SRLU_K1_TMEM=0 | tail -1 | tee -a $O/dbg_sweep.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k1t_kernel -c 1 -o $O/k1t_cfg2 -f python tools/k1_sweep.py 2 - > $O/ncu.log 2>&1; echo ncu rc=$?
