# A/B of design variants (libdialsort_<v>.so built with -D switches): c2 bench + phase times
for v in ${VARIANTS:-base}; do
  vv=$v; [ "$v" = base ] && vv=
  for c in ${CONFIGS:-c2}; do
    DIALSORT_LIB_VARIANT=$vv timeout 300 python bench.py --config $c --steps 300 --warmup 10 --no-cpu-baseline --no-e2e > gpurun_out/v.json 2>>gpurun_out/bench_err.log
    python -c "import json;d=json.load(open('gpurun_out/v.json'));print('variant [$v] $c', '%.4f ms'%d['ms_per_step'], 'frac %.3f'%d['roofline']['frac'])"
    [ "$v" = base ] && [ -z "$NOPHASE" ] && timeout 120 python tools/phase_times.py $c 2>&1 | tail -1
  done
done
