#!/bin/bash
# One GPU-box pass producing the evidence summarised under profiles/:
#   bench lines (C2 default with e2e + cpu_baseline, reference arm, C3, C5),
#   the ncu launch list of one C2 solve, --set full captures of the round
#   kernels (C2) and of one C5 k_pull.  Each ncu command runs only after the
#   same command exited 0 without ncu.  Usage: bash tools/profile.sh TAG
set -u
T=${1:-r01}
O=gpurun_out/prof_$T
mkdir -p $O
nvidia-smi > $O/nvidia_smi.txt 2>&1
python bench.py > $O/bench_c2.json 2> $O/bench_c2.err
python bench.py --impl reference --steps 3 --warmup 1 > $O/ref_c2.json 2> $O/ref_c2.err
python bench.py --config c3 --no-cpu-baseline > $O/bench_c3.json 2> $O/bench_c3.err
python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_c5.json 2> $O/bench_c5.err
export PUSHRANK_HOST_LOOP=1
B="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline"
if timeout 300 $B > $O/hostloop_c2.json 2>&1; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
    --log-file $O/launches_c2.csv $B > $O/ncu_launches.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_pull" \
    -s 60 -c 2 -o $O/full_c2 $B > $O/ncu_full_c2.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_scan|k_push" \
    -c 4 -o $O/sparse_c2 $B > $O/ncu_sparse_c2.log 2>&1
fi
B5="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --config c5"
if timeout 600 $B5 > $O/hostloop_c5.json 2>&1; then
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_pull" -s 30 -c 1 \
    -o $O/full_c5 $B5 > $O/ncu_full_c5.log 2>&1
fi
echo done
