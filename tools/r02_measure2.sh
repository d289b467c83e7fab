mkdir -p gpurun_out/r02
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/r02/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02/smoke.log 2>&1
timeout 1200 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02/bench_ref.json 2> gpurun_out/r02/bench_ref.err
timeout 1500 python bench.py --config c4 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/r02/bench_c4.json 2> gpurun_out/r02/bench_c4.err
