# HEAD validation: GPU suite (incl. the checked build), smoke, default bench line
mkdir -p gpurun_out/r02l
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02l/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/r02l/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02l/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r02l/smoke.log
timeout 1500 python bench.py > gpurun_out/r02l/bench.json 2> gpurun_out/r02l/bench.err; echo "rc=$?" >> gpurun_out/r02l/bench.err
echo done
