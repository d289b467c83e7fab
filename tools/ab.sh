# A/B quick bench: q <label> [env...]  (C3 10 iterations unless CFG set)
q() { lab=$1; shift; echo "== $lab"; env "$@" python bench.py --config ${CFG:-c3} --steps 1 --warmup 1 --iters ${ITERS:-10} --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['kernels_ms'])"; }
