set -x
mkdir -p gpurun_out/r2a
(nproc; free -g; lscpu; nvidia-smi; df -h /tmp /dev/shm) > gpurun_out/r2a/box.txt 2>&1
/usr/bin/time -v python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2a/c5.json 2> gpurun_out/r2a/c5.err
python bench.py --config c4 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2a/c4.json 2> gpurun_out/r2a/c4.err
python bench.py --config c4 --algo ifp1 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2a/c4_ifp1.json 2> gpurun_out/r2a/c4_ifp1.err
