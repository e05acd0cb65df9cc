#!/bin/bash
# A/B of library variants on the partitioned path: one NCCL rank at C5 and P emulated ranks.
# tools/part_ab.sh "base pb3" [P]
for v in $1; do
  if [ "$v" = base ]; then L=""; else L=$PWD/build/var/lib_$v.so; fi
  echo "== $v"
  PUSHRANK_LIB=$L PUSHRANK_PARTITIONED=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 1 --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('one rank', round(d['ms_per_step'],1), 'ms', d['rounds'], 'rounds')"
  PUSHRANK_LIB=$L tools/part_cost_sweep.sh 8 ${2:-8}
done
