# Baseline check: build, pytest -m gpu, short bench of every config
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
for c in ${CONFIGS:-c2 c3-zipf c3-sorted c3-hot1 c1 c5 c4}; do
  timeout 300 python bench.py --config $c --steps 100 --warmup 5 --no-cpu-baseline --no-e2e >> gpurun_out/bench_all.jsonl 2>> gpurun_out/bench_err.log
done
python - <<'PY'
import json
for l in open('gpurun_out/bench_all.jsonl'):
    d=json.loads(l); r=d['roofline']; st=d['step_roofline']
    print(d['config']['workload'][:42].ljust(42), '%.3e keys/s'%d['value'], '%.4f ms'%d['ms_per_step'], 'dom', r['kernel'], 'frac %.3f'%r['frac'], 'step %.3f'%st['frac_of_measured'])
PY
