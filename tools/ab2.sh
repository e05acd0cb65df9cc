#!/bin/bash
# A/B of library variants x environment settings on one box:
# tools/ab2.sh "lib:NAME=VAR=VAL,VAR=VAL ..." CONFIG [extra bench args]   (lib "base" = in-tree)
sets=$1; c=$2; shift 2
for s in $sets; do
  lib=${s%%:*}; rest=${s#*:}; name=${rest%%=*}; envs=$(echo "${rest#*=}" | tr ',' ' ')
  if [ "$lib" = base ]; then L=""; else L=$PWD/build/var/lib_$lib.so; fi
  env PUSHRANK_LIB=$L $envs timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --config $c "$@" > gpurun_out/v_${name}_$c.log 2>&1
done
