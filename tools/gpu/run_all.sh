set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
for c in c2 c1 c3-zipf c3-sorted c3-reverse c3-hot1 c5 c4; do
  timeout 300 python bench.py --config $c --steps 200 --warmup 10 --no-cpu-baseline --no-e2e >> gpurun_out/bench_all.jsonl 2>> gpurun_out/bench_err.log
done
timeout 300 python bench.py > gpurun_out/bench_default.jsonl 2>gpurun_out/bench_default.err; echo bench=$?
