python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
source tools/ab.sh
for r in 1 2; do ITERS=10 q e32; ITERS=10 q e16 HOLO_ADJ_E16=1; done
CFG=c2 ITERS=10 q c2-e32; CFG=c2 ITERS=10 q c2-e16 HOLO_ADJ_E16=1
