#!/bin/bash
# Final evidence pass of round 2: the -m gpu suite, the default C5 line, the
# other configs, IFP1, the partitioned path at one rank, the ncu launch list
# and per-section metrics of a C5 sweep.
O=gpurun_out/r2c; mkdir -p $O
nvidia-smi > $O/nvidia_smi.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/gputest.log 2>&1; echo "rc=$?" >> $O/gputest.log; tail -2 $O/gputest.log
timeout 900 python bench.py > $O/bench_c5.json 2> $O/bench_c5.err; cut -c1-200 $O/bench_c5.json
for c in c2 c3 c4; do
  timeout 600 python bench.py --config $c --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err
done
timeout 600 python bench.py --algo ifp1 --no-cpu-baseline --no-e2e > $O/bench_c5_ifp1.json 2> $O/bench_c5_ifp1.err
PUSHRANK_PARTITIONED=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29513 bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/part1_c5.json 2> $O/part1_c5.err
tools/ncu_sections.sh > $O/sections_c5.txt 2>&1
export PUSHRANK_HOST_LOOP=1
B5="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --config c5"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $O/launches_c5.csv $B5 > $O/ncu_launches.log 2>&1
python tools/launches.py $O/launches_c5.csv > $O/launches_c5.txt 2>&1
PUSHRANK_SORT_ROWS=1 timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_pull" -s 183 -c 1 -o $O/full_c5 $B5 > $O/ncu_full_c5.log 2>&1
python tools/ncu.py $O/full_c5.ncu-rep k_pull > $O/ncu_full_c5_k_pull.txt 2>&1
ncu -i $O/full_c5.ncu-rep --page raw --csv > $O/ncu_raw_full_c5.csv 2>/dev/null
rm -f $O/full_c5.ncu-rep
echo done
