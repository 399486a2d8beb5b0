# quick perf check: c2 + c3-zipf benches and phase timings (no tests)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for c in ${CONFIGS:-c2 c3-zipf}; do
  timeout 300 python bench.py --config $c --steps 300 --warmup 10 --no-cpu-baseline --no-e2e >> gpurun_out/bench_quick.jsonl 2>> gpurun_out/bench_err.log
  timeout 120 python tools/phase_times.py $c >> gpurun_out/phase_quick.txt 2>&1
done
python - <<'PY'
import json
for l in open('gpurun_out/bench_quick.jsonl'):
    d=json.loads(l); r=d['roofline']
    print(d['config']['workload'][:40].ljust(40), '%.3e'%d['value'], '%.4f ms'%d['ms_per_step'], r['kernel'], '%.3f'%r['frac'], 'step %.3f'%d['step_roofline']['frac_of_measured'], d['gpu_launches'])
PY
cat gpurun_out/phase_quick.txt
