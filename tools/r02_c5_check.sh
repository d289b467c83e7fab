mkdir -p gpurun_out/r02
python -m pytest tests/test_gpu_guard.py tests/test_gpu_fista.py tests/test_gpu_ops.py tests/test_gpu_parity_1024.py -x -q -p no:cacheprovider 2>&1 | tail -2
python bench.py --config c5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02/bench_c5.json 2> gpurun_out/r02/bench_c5.err
tail -1 gpurun_out/r02/bench_c5.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['kernels_ms'], d['clocks'])"
