#!/bin/bash
# Launch list of the partitioned path (one NCCL rank) next to the engine's, C3
O=${1:-gpurun_out/ncu_part}
mkdir -p $O
export PUSHRANK_PARTITIONED=1
timeout 900 ncu --target-processes all --metrics gpu__time_duration.sum --clock-control none -c 120 --csv \
  --log-file $O/part_c3.csv python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 \
  --master-port 29515 bench.py --steps 1 --warmup 1 --config c3 --no-e2e > $O/part_c3.log 2>&1
unset PUSHRANK_PARTITIONED
PUSHRANK_HOST_LOOP=1 PUSHRANK_GS_SECTIONS=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_pull -c 20 --csv \
  --log-file $O/engine_c3.csv python bench.py --steps 1 --warmup 0 --config c3 --no-e2e --no-cpu-baseline > $O/engine_c3.log 2>&1
