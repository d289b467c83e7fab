# Round-2 re-entry close: full GPU suite, smoke, cam bench line (with the reference parity leg)
mkdir -p gpurun_out/r02c
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02c/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/r02c/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02c/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r02c/smoke.log
timeout 900 python bench.py --config cam --steps 5 --warmup 3 > gpurun_out/r02c/bench_cam.json 2> gpurun_out/r02c/bench_cam.err
echo done
