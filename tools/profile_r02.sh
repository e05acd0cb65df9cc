#!/bin/bash
# Round-2 evidence pass on one GPU box (summarised under profiles/):
#   the -m gpu suite, bench lines (C5 default with e2e + cpu_baseline; the
#   reference arm; C2/C3/C4 and IFP1 C5), the partitioned path at one rank,
#   exchange volumes, the ncu launch list of one C5 solve and one --set full
#   capture of a C5 k_pull.  Each ncu command runs after the same command
#   exited 0 without ncu.  Usage: bash tools/profile_r02.sh TAG [skip-tests]
set -u
T=${1:-r02}
O=gpurun_out/prof_$T
mkdir -p $O
nvidia-smi > $O/nvidia_smi.txt 2>&1
if [ "${2:-}" != "skip-tests" ]; then
  timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/gputest.log 2>&1; echo "rc=$?" >> $O/gputest.log
fi
timeout 900 python bench.py > $O/bench_c5.json 2> $O/bench_c5.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/ref_c5.json 2> $O/ref_c5.err
for c in c2 c3 c4; do
  timeout 600 python bench.py --config $c --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err
done
timeout 600 python bench.py --algo ifp1 --no-cpu-baseline --no-e2e > $O/bench_c5_ifp1.json 2> $O/bench_c5_ifp1.err
PUSHRANK_PARTITIONED=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29513 bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/part1_c5.json 2> $O/part1_c5.err
timeout 900 python tools/exchange_volume.py c5 2 4 8 > $O/exchange_c5.jsonl 2> $O/exchange_c5.err
export PUSHRANK_HOST_LOOP=1
B5="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --config c5"
if timeout 600 $B5 > $O/hostloop_c5.json 2>&1; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
    --log-file $O/launches_c5.csv $B5 > $O/ncu_launches.log 2>&1
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_pull" -s 30 -c 1 \
    -o $O/full_c5 $B5 > $O/ncu_full_c5.log 2>&1
fi
echo done
