# full GPU parity suite, then short benches of the main configs
bash tools/gpu/run_tests.sh
rm -f gpurun_out/bench_all.jsonl
for c in ${CONFIGS:-c2 c3-zipf c5 c4}; do
  timeout 300 python bench.py --config $c --steps 100 --warmup 5 --no-cpu-baseline --no-e2e >> gpurun_out/bench_all.jsonl 2>> gpurun_out/bench_err.log
done
python - <<'PY'
import json
for l in open('gpurun_out/bench_all.jsonl'):
    d=json.loads(l); r=d['roofline']; st=d['step_roofline']
    print(d['config']['workload'][:42].ljust(42), '%.3e keys/s'%d['value'], '%.4f ms'%d['ms_per_step'], 'dom', r['kernel'], 'frac %.3f'%r['frac'], 'step %.3f'%st['frac_of_measured'])
PY
tail -3 gpurun_out/bench_err.log
