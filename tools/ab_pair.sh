cp variants/e_pair.so paper_1904_04884_b200/libholo_b200.so
timeout 600 python -m pytest tests/test_gpu_fista.py tests/test_gpu_ops.py tests/test_gpu_guard.py -x -q -p no:cacheprovider 2>&1 | grep -E "passed|failed|Error|assert" | tail -15
source tools/ab.sh
for r in 1 2; do ITERS=10 q c3_pair; ITERS=10 q c3_single HOLO_PROX_NOPAIR=1; done
