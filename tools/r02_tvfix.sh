# prox tvfix (54-row tiles, boundary-row TV terms from k_prox_tvfix): parity forced on every strip case, checked build, C3 A/B
mkdir -p gpurun_out/r02t
HOLO_PROX_TVFIX=1 timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02t/pytest_forced.log 2>&1; echo "rc=$?" >> gpurun_out/r02t/pytest_forced.log
HOLO_PROX_TVFIX=1 timeout 900 python tools/checked_solve.py > gpurun_out/r02t/normal.log 2>&1; echo "rc=$?" >> gpurun_out/r02t/normal.log
HOLO_PROX_TVFIX=1 HOLO_LIB_PATH=paper_1904_04884_b200/libholo_b200_checked.so timeout 900 python tools/checked_solve.py > gpurun_out/r02t/checked.log 2>&1; echo "rc=$?" >> gpurun_out/r02t/checked.log
HOLO_PROX_TVFIX=0 timeout 900 python tools/checked_solve.py > gpurun_out/r02t/off.log 2>&1; echo "rc=$?" >> gpurun_out/r02t/off.log
for r in 1 2; do
  timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02t/c3_fix_$r.json 2> gpurun_out/r02t/c3_fix_$r.err
  HOLO_PROX_TVFIX=0 timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02t/c3_nofix_$r.json 2> gpurun_out/r02t/c3_nofix_$r.err
done
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02t/pytest_default.log 2>&1; echo "rc=$?" >> gpurun_out/r02t/pytest_default.log
echo done
