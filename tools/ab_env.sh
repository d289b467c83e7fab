# A/B one library, env toggles: ab_env.sh "<label> <ENV=...>" ...
cp variants/*.so paper_1904_04884_b200/libholo_b200.so
python -m pytest tests/test_gpu_fista.py tests/test_gpu_guard.py -q -p no:cacheprovider 2>&1 | tail -1
source tools/ab.sh
for r in 1 2; do ITERS=10 q default; ITERS=10 q off HOLO_PROX_NOTT=1; done
