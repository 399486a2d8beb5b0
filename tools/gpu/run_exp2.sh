python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
VARIANTS="cv base cv base" MODES="0 1" KEXPR="partition_modes and 1048576 and 0" bash tools/gpu/run_part.sh
for c in c1 c2 c3-zipf; do
  timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e > gpurun_out/b_$c.json 2>gpurun_out/b_$c.err
  python -c "import json;d=json.load(open('gpurun_out/b_$c.json'));print('$c', d['ms_per_step'], d['roofline']['frac'], 'single', d.get('single_call',{}).get('ms_per_step') if d.get('single_call') else None, 'graph', (d.get('cuda_graph') or {}).get('ms_per_step'), d['verified'], d['verified_last_step'])"
done
