TLIM=1500 bash tools/gpu/run_tests.sh
timeout 300 python tools/kpc_ab.py 2>&1 | grep -v Warn
for c in c1 c2 c3-zipf c3-sorted; do
  timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e --steps 256 > gpurun_out/b_$c.json 2>gpurun_out/b_$c.err
  python -c "import json;d=json.load(open('gpurun_out/b_$c.json'));r=d['roofline'];print('$c', '%.5f'%d['ms_per_step'], '%.3f'%r['frac'], 'single', (d.get('single_call') or {}).get('ms_per_step'), d['verified'], d['verified_last_step'])"
done
