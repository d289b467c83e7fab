cp variants/e_pair.so paper_1904_04884_b200/libholo_b200.so
ncu --set full --import-source on --clock-control none -k regex:k_prox_strip -s 4 -c 1 -o gpurun_out/prox_pair python tools/run_solve.py 1024 1024 512 3 > gpurun_out/ncu_pair.log 2>&1
