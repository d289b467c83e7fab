source tools/ab.sh
for f in variants/*.so; do cp $f paper_1904_04884_b200/libholo_b200.so; python -m pytest tests/test_gpu_fista.py tests/test_gpu_guard.py -q -p no:cacheprovider 2>&1 | tail -1; done
for r in 1 2; do for f in variants/*.so; do cp $f paper_1904_04884_b200/libholo_b200.so; CFG=c5 ITERS=5 q "c5 $f"; done; done
