# quick perf check: c2 / zipf bench + phase stamps (phase build), then the given tests
for c in ${CONFIGS:-c2 c3-zipf}; do
  timeout 300 python bench.py --config $c --steps 300 --warmup 10 --no-cpu-baseline --no-e2e > gpurun_out/ab.json 2>>gpurun_out/bench_err.log
  python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('$c', '%.4f ms'%d['ms_per_step'], 'frac %.3f'%d['roofline']['frac'])"
  timeout 120 python tools/phase_times.py $c 2>&1 | tail -1
done
[ -n "$TESTS" ] && { timeout 900 python -m pytest $TESTS -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_gpu.log; }
tail -3 gpurun_out/bench_err.log
