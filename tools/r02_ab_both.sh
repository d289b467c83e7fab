# A/B of variants/*.so on both prox kinds: GPU tests, C5 passes (ncu per launch), then C3 prox (3 rounds)
bash tools/r02_ab_c5b.sh
for r in 1 2 3; do for f in variants/*.so; do cp $f paper_1904_04884_b200/libholo_b200.so; echo "== $r $f"; python bench.py --config c3 --steps 1 --warmup 1 --iters 10 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels_ms']; print(round(d['value']/1e9,3), round(d['ms_per_step'],2), 'prox', k['prox'])"; done; done
