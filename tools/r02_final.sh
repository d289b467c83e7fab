mkdir -p gpurun_out/r02
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02/pytest_gpu_final.log 2>&1; echo "rc=$?" >> gpurun_out/r02/pytest_gpu_final.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02/smoke_final.log 2>&1
timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/r02/bench_c3_final.json 2> gpurun_out/r02/bench_c3_final.err
