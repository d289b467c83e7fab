# A/B: per prebuilt library variant under variants/: GPU parity tests, then a quick C3 bench line (twice, interleaved)
T=${TESTS:-tests/test_gpu_fista.py tests/test_gpu_ops.py tests/test_gpu_guard.py}
for f in variants/*.so; do cp $f paper_1904_04884_b200/libholo_b200.so; echo "== $f"; python -m pytest $T -x -q -p no:cacheprovider 2>&1 | tail -1; done
for r in 1 2; do for f in variants/*.so; do cp $f paper_1904_04884_b200/libholo_b200.so; echo "== $r $f"; python bench.py --config ${CFG:-c3} --steps 1 --warmup 1 --iters ${ITERS:-10} --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e9,2), round(d['ms_per_step'],2), d['kernels_ms'])"; done; done
