#!/bin/bash
# ncu of the six section launches of one mid-solve C5 sweep (rows sorted at
# layout time, host-launched rounds): per-section L1/L2 request counts, hit
# rates, occupancy and stall mix.  Uses the pipe0 variant if present.
O=gpurun_out/sec; mkdir -p $O
export PUSHRANK_HOST_LOOP=1 PUSHRANK_SORT_ROWS=1
[ -n "$LIBV" ] && export PUSHRANK_LIB=$PWD/build/var/lib_$LIBV.so
B="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --config c5"
M=gpu__time_duration.sum,l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed,lts__t_requests_srcunit_tex.sum,lts__t_sectors_srcunit_tex.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld_lookup_hit.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,lts__t_sector_hit_rate.pct,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,sm__cycles_active.avg,smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct,smsp__warp_issue_stalled_barrier_per_warp_active.pct,smsp__warp_issue_stalled_lg_throttle_per_warp_active.pct,smsp__warp_issue_stalled_short_scoreboard_per_warp_active.pct,smsp__warp_issue_stalled_wait_per_warp_active.pct,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed
timeout 1200 ncu --metrics $M --clock-control none -k regex:"k_pull" -s 180 -c 6 --csv --log-file $O/sections.csv $B > $O/ncu.log 2>&1
python - <<'PY'
import csv, collections
rows=list(csv.reader(open('gpurun_out/sec/sections.csv')))
hi=[i for i,r in enumerate(rows) if r and r[0]=="ID"][0]
hdr=rows[hi]; data=rows[hi+1:]
ix={h:i for i,h in enumerate(hdr)}
per=collections.OrderedDict()
for r in data:
    per.setdefault(r[ix["ID"]],{})[r[ix["Metric Name"]]]=(r[ix["Metric Value"]],r[ix["Metric Unit"]])
names=sorted({k for v in per.values() for k in v})
print("metric".ljust(80)+" ".join(f"{'sec'+str(i):>14s}" for i in range(len(per))))
for n in names:
    print(n.ljust(80)+" ".join(f"{v.get(n,('',''))[0]:>14s}" for v in per.values()))
PY
