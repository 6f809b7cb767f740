mkdir -p /tmp/bin && nvcc -cudart shared -DSRLU_LU_TRACE -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -std=c++17 tools/lu_trace.cu paper_1601_04280_b200/csrc/abi.cu -o /tmp/bin/lu_trace || exit 1
for b2 in 1 0; do for s in "262144 220" "1048576 120"; do echo "b2=$b2 $s: $(SRLU_LU_B2=$b2 /tmp/bin/lu_trace $s | tail -1)"; done; done
