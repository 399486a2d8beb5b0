# GPU parity tests (all, or the files/-k given in TESTS), then smoke
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -2 gpurun_out/smoke.log
timeout ${TLIM:-1500} python -m pytest ${TESTS:-tests} -m gpu -x -q ${PYARGS} > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -15 gpurun_out/pytest_gpu.log
