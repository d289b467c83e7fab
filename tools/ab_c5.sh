source tools/ab.sh
python -m pytest tests/test_gpu_fista.py -q -p no:cacheprovider -k "shapes_and_inner or edge_shapes" 2>&1 | tail -1
HOLO_PASS_LEN=10 python -m pytest tests/test_gpu_fista.py -q -p no:cacheprovider -k "shapes_and_inner or edge_shapes" 2>&1 | tail -1
for r in 1 2; do CFG=c5 ITERS=5 q c5_default; CFG=c5 ITERS=5 q c5_pass10 HOLO_PASS_LEN=10; CFG=c5 ITERS=5 q c5_pass8 HOLO_PASS_LEN=8; done
