# ncu --set full of the mixed-radix kernels (gfft.cu) on a 1000x1000x64 solve, then the final full GPU suite
mkdir -p gpurun_out/r02g
timeout 300 python tools/time_general.py 1000 1000 64 3 > gpurun_out/r02g/plain.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_grows|k_gcols|k_gadj|k_gfwd" -s 8 -c 4 -o gpurun_out/r02g/gen python tools/time_general.py 1000 1000 64 3 > gpurun_out/r02g/ncu.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02g/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/r02g/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02g/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r02g/smoke.log
echo done
