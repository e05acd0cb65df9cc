#!/bin/bash
# A/B of the index upload at C5 on one box: adaptive split against static
# splits and fewer host threads (a slow host).  tools/upload_ab.sh [steps]
STEPS=${1:-3}
for v in "adaptive" "PUSHRANK_UPLOAD_HOSTFRAC=0.9" "PUSHRANK_UPLOAD_HOSTFRAC=0.6" "PUSHRANK_UPLOAD_HOSTFRAC=0" \
         "PUSHRANK_UPLOAD_THREADS=4" "PUSHRANK_UPLOAD_THREADS=4 PUSHRANK_UPLOAD_HOSTFRAC=0.9"; do
  echo "== $v"
  if [ "$v" = adaptive ]; then v=""; fi
  env $v PUSHRANK_TIMING=1 python tools/e2e_phases.py c5 $STEPS 2>&1 | grep -E "^\[upload\]|^step" | tail -$((2*STEPS))
done
