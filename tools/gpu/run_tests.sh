# GPU parity tests (all, or the files given in TESTS, filtered by the -k expression KEXPR), then smoke
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -2 gpurun_out/smoke.log
if [ -n "$KEXPR" ]; then
  timeout ${TLIM:-1500} python -m pytest ${TESTS:-tests} -m gpu -x -q ${PYARGS} -k "$KEXPR" > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
else
  timeout ${TLIM:-1500} python -m pytest ${TESTS:-tests} -m gpu -x -q ${PYARGS} > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
fi
tail -15 gpurun_out/pytest_gpu.log
