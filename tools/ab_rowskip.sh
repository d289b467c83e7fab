# Sparsity-aware forward (row skipping) A/B: GPU tests, C3 / C4 quick bench with and without HOLO_ROWSKIP, a sparse scene
python -m pytest tests/test_gpu_fista.py tests/test_gpu_ops.py tests/test_gpu_guard.py -q -p no:cacheprovider 2>&1 | grep -E "passed|failed|Error|assert" | tail -15
source tools/ab.sh
for r in 1 2; do ITERS=10 q c3_dense; ITERS=10 q c3_rowskip HOLO_ROWSKIP=1; done
CFG=c4 ITERS=5 q c4_dense; CFG=c4 ITERS=5 q c4_rowskip HOLO_ROWSKIP=1
for r in 1 2; do echo "== sparse dense"; python tools/run_solve.py 1024 1024 256 20; echo "== sparse rowskip"; HOLO_ROWSKIP=1 python tools/run_solve.py 1024 1024 256 20; done
