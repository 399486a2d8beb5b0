python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
for c in c2 c3-zipf c3-sorted c1; do
  timeout 300 python bench.py --config $c --steps 300 --warmup 10 --no-cpu-baseline --no-e2e >> gpurun_out/bench_fused2.jsonl 2>> gpurun_out/bench_err.log
done
timeout 120 python tools/phase_times.py c2 > gpurun_out/phase_fused2.txt 2>&1
timeout 120 python tools/phase_times.py c3-zipf >> gpurun_out/phase_fused2.txt 2>&1
cat gpurun_out/phase_fused2.txt
