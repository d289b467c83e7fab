# Round-2 measurement batch (one GPU): launcher + NCCL single-rank path, C3 default line,
# ncu launch list of a 2-step C3 bench, C2 / C5 lines.
mkdir -p gpurun_out/r02
HOLO_SELF_LAUNCH=1 HOLO_NCCL_SINGLE_RANK=1 timeout 900 python bench.py --gpus 1 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r02/launcher_nccl1.json 2> gpurun_out/r02/launcher_nccl1.err
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r02/bench_c3.json 2> gpurun_out/r02/bench_c3.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/r02/launches_c3.csv python bench.py --steps 1 --warmup 3 --iters 10 --no-cpu-baseline --no-e2e > gpurun_out/r02/ncu_launch.log 2>&1
timeout 900 python bench.py --config c2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02/bench_c2.json 2> gpurun_out/r02/bench_c2.err
timeout 900 python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r02/bench_c5.json 2> gpurun_out/r02/bench_c5.err
