for f in variants/*.so; do cp $f paper_1904_04884_b200/libholo_b200.so; echo "== $f"; python -m pytest tests/test_gpu_ops.py -x -q -p no:cacheprovider 2>&1 | tail -1; done
source tools/ab.sh
for r in 1 2; do for f in variants/*.so; do cp $f paper_1904_04884_b200/libholo_b200.so; ITERS=10 q "c3 $f"; done; done
for f in variants/*.so; do cp $f paper_1904_04884_b200/libholo_b200.so; CFG=c4 ITERS=5 q "c4 $f"; done
