# Round-2 re-entry: GPU suite, C3 bench line, compute-sanitizer over every kernel family
mkdir -p gpurun_out/r02s
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/r02s/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02s/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/r02s/pytest_gpu.log
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/r02s/bench_c3.json 2> gpurun_out/r02s/bench_c3.err
for tool in memcheck synccheck racecheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_solve.py \
    > gpurun_out/r02s/san_${tool}.log 2>&1
  echo "rc=$?" >> gpurun_out/r02s/san_${tool}.log
done
echo done
