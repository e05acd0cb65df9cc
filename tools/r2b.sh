#!/bin/bash
# Round-2 (second half) evidence run at C5 with the 6-section default:
# forced-C5 parity test, the full-size C5 parity script, the default bench
# line, IFP1, and the partitioned path at one rank.
O=gpurun_out/r2b; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "forced_c5 or c5_full_size or gauss_seidel" > $O/pytest_c5.log 2>&1; tail -2 $O/pytest_c5.log
timeout 600 python bench.py > $O/bench_c5.json 2> $O/bench_c5.err; cut -c1-300 $O/bench_c5.json
timeout 300 python bench.py --algo ifp1 --no-cpu-baseline --no-e2e > $O/bench_c5_ifp1.json 2>> $O/bench_c5.err
PUSHRANK_PARTITIONED=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 5 --warmup 3 --no-cpu-baseline > $O/part1_c5.json 2> $O/part1_c5.err
(cd tests && timeout 3000 python full_size_parity.py c5 --out ../$O/parity_c5.json > ../$O/parity_c5.log 2>&1); tail -2 $O/parity_c5.log
