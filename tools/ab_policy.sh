#!/bin/bash
# AUTO policy sweep (push below this fraction of the dense work) and IFP1 lines
O=${1:-gpurun_out/ab_policy}
mkdir -p $O
for c in c2 c4 c3; do
  for ps in 0.02 0.05 0.1 0.2; do
    timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --config $c --push-switch $ps > $O/${c}_ps$ps.json 2> $O/${c}_ps$ps.err
  done
  timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --config $c --algo ifp1 > $O/${c}_ifp1.json 2> $O/${c}_ifp1.err
done
