# Round-2 re-entry closing measurements: GPU suite (incl. general plane sides), smoke, C3 line, launch list
mkdir -p gpurun_out/r02z
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02z/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/r02z/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02z/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r02z/smoke.log
timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/r02z/bench_c3.json 2> gpurun_out/r02z/bench_c3.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r02z/bench_c3_reference.json 2> gpurun_out/r02z/bench_c3_reference.err
timeout 600 python bench.py --steps 1 --warmup 3 --iters 10 --no-cpu-baseline --no-e2e > gpurun_out/r02z/launches_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/r02z/launches.csv python bench.py --steps 1 --warmup 3 --iters 10 --no-cpu-baseline --no-e2e > gpurun_out/r02z/launches.log 2>&1
echo done
