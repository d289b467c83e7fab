for r in 1 2; do for f in variants/*.so; do cp $f paper_1904_04884_b200/libholo_b200.so; echo "== $f"; python tools/time_prox_op.py 64 5 20; done; done
