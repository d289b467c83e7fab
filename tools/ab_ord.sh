# A/B the interior-first region order of the T = 5 main prox launch (HOLO_PROX_NOORD=1: off)
python -m pytest tests/test_gpu_fista.py tests/test_gpu_guard.py tests/test_gpu_parity_1024.py -q -p no:cacheprovider 2>&1 | tail -2
source tools/ab.sh
for r in 1 2 3; do ITERS=10 q ord; ITERS=10 q noord HOLO_PROX_NOORD=1; done
CFG=c2 ITERS=10 q c2-ord; CFG=c2 ITERS=10 q c2-noord HOLO_PROX_NOORD=1
