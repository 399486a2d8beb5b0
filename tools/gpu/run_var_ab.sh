# A/B of library variants (VARIANTS, "base" = libdialsort.so) on bench configs (CONFIGS), batch and single call
for v in ${VARIANTS:-base}; do
  vv=$v; [ "$v" = base ] && vv=
  for c in ${CONFIGS:-c2 c3-zipf}; do
    for b in ${BATCHES:-32 1}; do
      DIALSORT_LIB_VARIANT=$vv timeout 300 python bench.py --config $c --steps ${STEPS:-320} --warmup 32 --batch $b --no-cpu-baseline --no-e2e > gpurun_out/v.json 2>>gpurun_out/bench_err.log
      python -c "import json;d=json.load(open('gpurun_out/v.json'));print('variant [$v] $c batch=$b', '%.4f ms'%d['ms_per_step'], 'best %.4f'%d['reps']['best_ms_per_step'], 'frac %.3f'%d['roofline']['frac'], d['verified_last_step'])"
    done
  done
done
tail -2 gpurun_out/bench_err.log
