source tools/ab.sh
for r in 1 2; do for f in variants/*.so; do cp $f paper_1904_04884_b200/libholo_b200.so; ITERS=10 q "c3 $f"; done; done
