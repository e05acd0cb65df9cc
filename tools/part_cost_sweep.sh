#!/bin/bash
# Partition row-cost sweep with emulated ranks: tools/part_cost_sweep.sh "8 16 24" [P] [config]
for rc in $1; do
  PUSHRANK_PART_ROW_COST=$rc timeout 600 python tools/emulated_scaling.py ${3:-c5} ${2:-8} 2>/dev/null | RC=$rc python -c "
import json, os, sys
for l in sys.stdin:
    d = json.loads(l)
    print('row_cost', os.environ['RC'], 'P', d['parts'], 'rounds', d['rounds'], d['rank_kernel_ms_total'], 'modelled', d['modelled_solve_ms'])
"
done
