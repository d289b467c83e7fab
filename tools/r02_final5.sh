# Round-2 closing measurements after tvfix (54-row prox tiles): GPU suite, smoke, C3/C2/C5/C4 lines, reference arm, launch list
mkdir -p gpurun_out/r02y
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02y/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/r02y/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02y/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r02y/smoke.log
timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/r02y/bench_c3.json 2> gpurun_out/r02y/bench_c3.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r02y/bench_c3_reference.json 2> gpurun_out/r02y/bench_c3_reference.err
timeout 900 python bench.py --config c2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02y/bench_c2.json 2> gpurun_out/r02y/bench_c2.err
timeout 900 python bench.py --config c5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02y/bench_c5.json 2> gpurun_out/r02y/bench_c5.err
timeout 1200 python bench.py --config c4 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r02y/bench_c4.json 2> gpurun_out/r02y/bench_c4.err
timeout 600 python bench.py --steps 1 --warmup 3 --iters 10 --no-cpu-baseline --no-e2e > gpurun_out/r02y/launches_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/r02y/launches.csv python bench.py --steps 1 --warmup 3 --iters 10 --no-cpu-baseline --no-e2e > gpurun_out/r02y/launches.log 2>&1
echo done
