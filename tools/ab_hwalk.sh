cp variants/d_hwalk.so paper_1904_04884_b200/libholo_b200.so
python -m pytest tests/test_gpu_fista.py tests/test_gpu_ops.py tests/test_gpu_guard.py tests/test_gpu_parity_1024.py -q -p no:cacheprovider 2>&1 | grep -E "passed|failed|Error|assert" | tail -15
source tools/ab.sh
for r in 1 2; do ITERS=10 q c3_hwalk; ITERS=10 q c3_tiled HOLO_PROX_NOHWALK=1; done
