#!/bin/bash
# A/B of library variants on one box: tools/ab.sh "v1 v2 ..." "c2 c3" [extra bench args]
# variant "base" = the in-tree library; others = build/var/lib_<v>.so
for v in $1; do
  if [ "$v" = base ]; then L=""; else L=$PWD/build/var/lib_$v.so; fi
  for c in $2; do
    PUSHRANK_LIB=$L timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --config $c $3 > gpurun_out/v_${v}_$c.log 2>&1
  done
done
