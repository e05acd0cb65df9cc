mkdir -p gpurun_out/s4
export PUSHRANK_LIB=$PWD/build/var/lib_ubench.so
export PUSHRANK_SORT_ROWS=1
for H in 4096 16384 32768; do PR_UB_H=$H UB_BPS=4 timeout 300 python tools/ubench.py c5 2,7,8 >> gpurun_out/s4/ub.txt 2>&1; done
for H in 2048 4096 6144; do PR_UB_H=$H UB_BPS=4 timeout 300 python tools/ubench.py c5 9 >> gpurun_out/s4/ub.txt 2>&1; done
unset PUSHRANK_LIB PUSHRANK_SORT_ROWS
PUSHRANK_TIMING=1 timeout 600 python tools/e2e_phases.py c5 3 > gpurun_out/s4/e2e.txt 2>&1
