# GPU parity tests, c4 bench, ncu capture of k_part_scatter (iteration loop for the partition kernels)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu.log
for c in ${CONFIGS:-c4}; do timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --no-e2e >> gpurun_out/bench_quick.jsonl; done
[ -n "$NOPROF" ] || bash tools/gpu/run_prof_c4.sh
