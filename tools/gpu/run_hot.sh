python -c "import __graft_entry__ as g; g.build()" >/dev/null
timeout 900 python -m pytest tests/test_gpu.py -m gpu -x -q -k "hot or overflow or skew or c3 or c2 or c1 or format or boundaries" 2>&1 | tail -3
timeout 600 python tools/skew_scale.py
for c in c2 c3-zipf c3-hot1; do
  timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e --steps 256 > gpurun_out/b_$c.json 2>gpurun_out/b_$c.err
  python -c "import json;d=json.load(open('gpurun_out/b_$c.json'));r=d['roofline'];print('$c', '%.5f'%d['ms_per_step'], '%.3f'%r['frac'], 'single', (d.get('single_call') or {}).get('ms_per_step'), d['verified'], d['verified_last_step'])"
done
