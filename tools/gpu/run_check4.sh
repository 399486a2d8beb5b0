# full GPU tests + bench lines of the fused-step configs (and c4)
TLIM=1500 bash tools/gpu/run_tests.sh
for c in c2 c3-zipf c3-sorted c3-hot1 c1 c4; do
  timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e --steps ${STEPS:-256} > gpurun_out/b_$c.json 2>gpurun_out/b_$c.err
  python -c "import json;d=json.load(open('gpurun_out/b_$c.json'));r=d['roofline'];print('$c', '%.5f'%d['ms_per_step'], r['kernel'], '%.3f'%r['frac'], 'single', (d.get('single_call') or {}).get('ms_per_step'), r.get('kernels_ms') if '$c'=='c4' else '', d['verified'], d['verified_last_step'])"
done
