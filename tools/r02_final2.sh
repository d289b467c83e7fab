# Round-2 closing measurements: full GPU suite, smoke, driver-style bench lines, ncu launch list and one
# --set full capture of each main C3 kernel class (traffic) -- run one after another, no ncu on bench numbers
mkdir -p gpurun_out/r02f
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02f/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/r02f/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02f/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r02f/smoke.log
timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/r02f/bench_c3.json 2> gpurun_out/r02f/bench_c3.err
timeout 900 python bench.py --config c2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02f/bench_c2.json 2> gpurun_out/r02f/bench_c2.err
timeout 1200 python bench.py --config c4 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r02f/bench_c4.json 2> gpurun_out/r02f/bench_c4.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/r02f/launches.csv python bench.py --steps 1 --warmup 3 --iters 10 --no-cpu-baseline --no-e2e > gpurun_out/r02f/launches.log 2>&1
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:"k_prox_strip|k_adj_cols|k_fwd_cols_staged|k_fft_rows" -s 40 -c 5 -o gpurun_out/r02f/full python bench.py --steps 1 --warmup 1 --iters 10 --no-cpu-baseline --no-e2e > gpurun_out/r02f/full.log 2>&1
echo done
