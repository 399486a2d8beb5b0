python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu.py -x -q -k "c1 or small_cluster or random_sweep or universe_bound or unaligned or in_place or empty or key_range or argument or paper_worked or heavy_skew or hot_key" > gpurun_out/t_small.log 2>&1
for sm in 1 0; do
  DIALSORT_SMALL=$sm timeout 300 python bench.py --config c1 --steps 320 --warmup 32 --no-cpu-baseline --no-e2e 2>/dev/null | grep '^{' | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('c1 small=$sm single', round(d['single_call']['ms_per_step']*1000,2), 'graph', round(d['cuda_graph']['ms_per_step']*1000,2), d['verified'])" >> gpurun_out/ab.log
done
timeout 900 python bench.py --grid > gpurun_out/r02s2_paper_grid.jsonl 2> gpurun_out/grid.err; echo grid=$? >> gpurun_out/ab.log
