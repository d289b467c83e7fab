# column-pair-blocked forward exchange: GPU tests, then C3 10-iteration A/B against the row-major path (env switch)
python -m pytest tests/test_gpu_fista.py tests/test_gpu_ops.py tests/test_gpu_parity_1024.py tests/test_gpu_prox_order.py -x -q -p no:cacheprovider 2>&1 | tail -2
source tools/ab.sh
for r in 1 2 3; do ITERS=10 q blocked; ITERS=10 q rowmajor HOLO_FWD_ROWMAJOR=1; done
