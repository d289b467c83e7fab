# sustained (power-capped) A/B of variants/*.so: C3 bench lines at 100 iterations, 5 timed solves each, 3 alternating rounds
for r in 1 2 3; do for f in variants/*.so; do cp $f paper_1904_04884_b200/libholo_b200.so; echo "== $r $f"
  python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels_ms']; print(round(d['value']/1e9,3), round(d['ms_per_step'],1), 'prox', k['prox'], 'clk', d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done; done
