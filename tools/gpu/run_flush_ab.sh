python -c "import __graft_entry__ as g; g.build()" >/dev/null
for v in base fshfl fnots base fshfl fnots; do
  vv=$v; [ $v = base ] && vv=
  DIALSORT_LIB_VARIANT=$vv timeout 300 python bench.py --config c2 --steps 256 --warmup 32 --no-cpu-baseline --no-e2e > gpurun_out/v.json 2>>gpurun_out/bench_err.log
  python -c "import json;d=json.load(open('gpurun_out/v.json'));print('[$v] c2', '%.4f'%d['ms_per_step'], 'single %.4f'%d['single_call']['ms_per_step'], d['verified'])"
done
