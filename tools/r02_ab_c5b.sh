for f in variants/*.so; do cp $f paper_1904_04884_b200/libholo_b200.so; echo "== $f"; python -m pytest tests/test_gpu_guard.py tests/test_gpu_fista.py -x -q -p no:cacheprovider 2>&1 | tail -1; done
bash tools/ab_prox_ncu.sh
