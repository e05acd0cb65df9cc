#!/bin/bash
# A/B of environment settings on one box: tools/ab_env.sh CONFIG "NAME=VAR=VAL[,VAR=VAL] ..." [extra bench args]
c=$1; shift; sets=$1; shift
for s in $sets; do
  name=${s%%=*}; rest=${s#*=}
  envs=$(echo "$rest" | tr ',' ' ')
  env $envs timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --config $c "$@" > gpurun_out/v_${name}_$c.log 2>&1
done
