# full GPU tests + the default bench line (c2) and c1 with the CUDA-graph leg
TLIM=1200 bash tools/gpu/run_tests.sh
for c in c2 c1; do
  timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/b_$c.json 2>gpurun_out/b_$c.err
  python -c "import json;d=json.load(open('gpurun_out/b_$c.json'));print('$c', d['ms_per_step'], d['roofline']['frac'], 'single', d.get('single_call',{}).get('ms_per_step') if d.get('single_call') else None, 'graph', d.get('cuda_graph'))"
done
