# GPU parity tests, then the quick perf check
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
bash tools/gpu/run_quick.sh
timeout 120 python tools/phase_times.py c2 > gpurun_out/phase_cta.txt 2>&1
grep -A1 "rep 3" gpurun_out/phase_cta.txt
