# One --set full source capture of the engine's main prox launch (FAST T = 5, interior-first order), C3 planes
mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none -k regex:"k_prox_strip" -s 4 -c 3 -o gpurun_out/prox_ord python tools/run_solve.py 1024 1024 512 3 > gpurun_out/ncu_prox_ord.log 2>&1
echo rc=$? >> gpurun_out/ncu_prox_ord.log
