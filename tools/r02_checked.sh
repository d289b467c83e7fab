# bounds-checked build vs normal build (compute-sanitizer substitute)
mkdir -p gpurun_out/r02c
timeout 900 python tools/checked_solve.py > gpurun_out/r02c/normal.log 2>&1; echo "rc=$?" >> gpurun_out/r02c/normal.log
HOLO_LIB_PATH=paper_1904_04884_b200/libholo_b200_checked.so timeout 900 python tools/checked_solve.py > gpurun_out/r02c/checked.log 2>&1; echo "rc=$?" >> gpurun_out/r02c/checked.log
timeout 1200 python -m pytest tests/test_gpu_checked.py tests/test_gpu_guard.py tests/test_gpu_plane_skip.py -q -p no:cacheprovider > gpurun_out/r02c/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02c/pytest.log
echo done
