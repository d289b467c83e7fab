cp variants/d_split.so paper_1904_04884_b200/libholo_b200.so
python -m pytest tests/test_gpu_guard.py tests/test_gpu_fista.py tests/test_gpu_ops.py "tests/test_gpu_parity_1024.py" -x -q -p no:cacheprovider 2>&1 | tail -3
bash tools/ab_prox_ncu.sh
