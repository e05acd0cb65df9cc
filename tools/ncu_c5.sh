#!/bin/bash
# ncu --set full of one mid-solve C5 k_pull launch (host-launched rounds:
# ncu cannot profile kernels inside conditional graphs).  Usage: tools/ncu_c5.sh TAG [config]
T=${1:-r02}; C=${2:-c5}
O=gpurun_out/ncu_$T; mkdir -p $O
export PUSHRANK_HOST_LOOP=1
B="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --config $C"
if timeout 600 $B > $O/hostloop_$C.json 2>&1; then
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_pull" -s ${SKIP:-30} -c ${COUNT:-1} \
    -o $O/full_$C $B > $O/ncu_full_$C.log 2>&1
  echo "ncu rc=$?"
fi
