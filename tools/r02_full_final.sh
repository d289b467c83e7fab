# final-state ncu --set full capture of each main C3 kernel class (bench hologram, 10 iterations)
mkdir -p gpurun_out/r02f
timeout 600 python bench.py --steps 1 --warmup 1 --iters 10 --no-cpu-baseline --no-e2e > gpurun_out/r02f/plain.log 2>&1 && \
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:"k_prox_strip|k_adj_cols|k_fwd_cols_staged|k_fft_rows" -s 40 -c 5 -o gpurun_out/r02f/full python bench.py --steps 1 --warmup 1 --iters 10 --no-cpu-baseline --no-e2e > gpurun_out/r02f/ncu.log 2>&1
echo done
