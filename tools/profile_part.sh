#!/bin/bash
# Partitioned path evidence (one NCCL rank, fused exchange): bench lines for
# C2/C3/C5 and one ncu --set full capture of k_part_pull at C3.  Each ncu
# command runs only after the same command exited 0 without ncu.
O=${1:-gpurun_out/prof_part}
mkdir -p $O
export PUSHRANK_PARTITIONED=1
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1"
for c in c2 c3; do
  timeout 600 $R --master-port 29521 bench.py --steps 5 --warmup 3 --config $c > $O/part_$c.json 2> $O/part_$c.err
done
B="$R --master-port 29522 bench.py --steps 1 --warmup 1 --config c3 --no-e2e"
if timeout 600 $B > $O/part_c3_short.json 2>&1; then
  timeout 900 ncu --target-processes all --set full --clock-control none --import-source on -k regex:k_part_pull \
    -s 20 -c 1 -o $O/full_part_c3 $B > $O/ncu_full_part_c3.log 2>&1
fi
