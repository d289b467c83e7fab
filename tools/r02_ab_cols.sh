# column-pass A/B of variants/*.so: GPU tests, then C3 (10 iterations) kernel ms, 2 interleaved rounds
for f in variants/*.so; do cp $f paper_1904_04884_b200/libholo_b200.so; echo "== $f"; python -m pytest tests/test_gpu_fista.py tests/test_gpu_ops.py -x -q -p no:cacheprovider 2>&1 | tail -1; done
for r in 1 2; do for f in variants/*.so; do cp $f paper_1904_04884_b200/libholo_b200.so; echo "== $r $f"
  python bench.py --config c3 --steps 1 --warmup 1 --iters 10 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels_ms']; print('c3', round(d['value']/1e9,3), 'adj_cols', k['adj_cols'], 'fwd_cols', k['fwd_cols'])"
done; done
