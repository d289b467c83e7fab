# plane-skipping: parity tests, A/B on a sparse-slab scene, C3 overhead A/B
mkdir -p gpurun_out/r02k
timeout 900 python -m pytest tests/test_gpu_plane_skip.py -q -p no:cacheprovider > gpurun_out/r02k/pytest_skip.log 2>&1; echo "rc=$?" >> gpurun_out/r02k/pytest_skip.log
timeout 900 python tools/time_plane_skip.py 20 > gpurun_out/r02k/time_skip.log 2>&1; echo "rc=$?" >> gpurun_out/r02k/time_skip.log
for r in 1 2; do
  timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02k/c3_skip_$r.json 2> gpurun_out/r02k/c3_skip_$r.err
  HOLO_NO_PLANE_SKIP=1 timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02k/c3_noskip_$r.json 2> gpurun_out/r02k/c3_noskip_$r.err
done
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02k/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/r02k/pytest_gpu.log
echo done
