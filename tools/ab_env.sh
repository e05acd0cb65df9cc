#!/bin/bash
# A/B of an environment switch: tools/ab_env.sh OUTDIR VAR "v1 v2" "c2 c3 ..." [extra bench args]
O=$1; V=$2
mkdir -p $O
for c in $4; do
  for v in $3; do
    env $V=$v timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --config $c $5 \
      > $O/${c}_$v.json 2> $O/${c}_$v.err
  done
done
