mkdir -p gpurun_out/v19
for v in base s16; do
  if [ "$v" = base ]; then L=""; else L=$PWD/build/var/lib_$v.so; fi
  for so in 0 1; do
    PUSHRANK_LIB=$L PUSHRANK_SORT_ROWS=$so timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --config c5 > gpurun_out/v19/c5_${v}_sort$so.json 2> gpurun_out/v19/c5_${v}_sort$so.err
  done
done
PUSHRANK_SORT_ROWS=1 timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --config c3 > gpurun_out/v19/c3_base_sort1.json 2> gpurun_out/v19/c3_base_sort1.err
PUSHRANK_LIB=$PWD/build/var/lib_s16.so PUSHRANK_SORT_ROWS=1 timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --config c3 > gpurun_out/v19/c3_s16_sort1.json 2> gpurun_out/v19/c3_s16_sort1.err
