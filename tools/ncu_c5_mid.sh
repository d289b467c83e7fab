# --set full source capture of one middle pass of the C5-shaped multi-pass prox (T = 20)
mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none -k regex:"k_prox_strip" -s 4 -c 3 -o gpurun_out/c5_mid python tools/run_solve.py 1024 1024 512 2 20 > gpurun_out/ncu_c5_mid.log 2>&1
echo rc=$? >> gpurun_out/ncu_c5_mid.log
