mkdir -p tools/bin && nvcc -cudart shared -DSRLU_LU_TRACE -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -std=c++17 tools/lu_trace.cu paper_1601_04280_b200/csrc/abi.cu -o tools/bin/lu_trace || exit 1
for pf in 0 1 2 4 8; do for s in "262144 220" "1048576 120" "65536 550" "65536 550 c"; do echo "pf=$pf $s: $(SRLU_LU_L2PF=$pf tools/bin/lu_trace $s | tail -1)"; done; done
