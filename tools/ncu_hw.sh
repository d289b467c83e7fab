cp variants/d_hwalk.so paper_1904_04884_b200/libholo_b200.so
ncu --set full --import-source on --clock-control none -k regex:k_prox_strip -s 4 -c 1 -o gpurun_out/prox_hwalk python tools/run_solve.py 1024 1024 512 3 > gpurun_out/ncu_hw.log 2>&1
HOLO_PROX_NOHWALK=1 ncu --set full --import-source on --clock-control none -k regex:k_prox_strip -s 4 -c 1 -o gpurun_out/prox_tiled python tools/run_solve.py 1024 1024 512 3 >> gpurun_out/ncu_hw.log 2>&1
