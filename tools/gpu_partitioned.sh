# Partitioned-path checks on one GPU: CUDA local-step tests, the partitioned bench at one NCCL rank
# (PUSHRANK_PARTITIONED=1) for C2/C3/C5, and two gloo ranks sharing the GPU (functional).
mkdir -p ${OUT:-gpurun_out/part}
timeout 600 python -m pytest tests/test_gpu_distributed.py -x -q > ${OUT:-gpurun_out/part}/pytest.log 2>&1; echo pytest=$? >> ${OUT:-gpurun_out/part}/pytest.log
for c in c2 c3; do
PUSHRANK_PARTITIONED=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --steps 5 --warmup 3 --config $c > ${OUT:-gpurun_out/part}/part1_$c.json 2> ${OUT:-gpurun_out/part}/part1_$c.err
done
PUSHRANK_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --steps 3 --warmup 3 --config c2 > ${OUT:-gpurun_out/part}/gloo2_c2.json 2> ${OUT:-gpurun_out/part}/gloo2_c2.err
PUSHRANK_PARTITIONED=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29513 bench.py --steps 2 --warmup 3 --config c5 > ${OUT:-gpurun_out/part}/part1_c5.json 2> ${OUT:-gpurun_out/part}/part1_c5.err
PUSHRANK_FUSED=0 PUSHRANK_PARTITIONED=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29514 bench.py --steps 5 --warmup 3 --config c3 > ${OUT:-gpurun_out/part}/part1_c3_gathered.json 2> ${OUT:-gpurun_out/part}/part1_c3_gathered.err
