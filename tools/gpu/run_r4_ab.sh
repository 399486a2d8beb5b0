# radix pass variants (VARIANTS: library variants, base = libdialsort.so) on c5
for v in ${VARIANTS:-base}; do
  DIALSORT_LIB_VARIANT=$( [ $v = base ] && echo "" || echo $v ) timeout 300 python bench.py --config c5 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r4.json 2>>gpurun_out/bench_err.log
  python -c "import json;d=json.load(open('gpurun_out/r4.json'));r=d['roofline'];print('$v', '%.4f ms'%d['ms_per_step'], 'pass %.4f'%r['avg_ms'], 'frac %.3f'%r['frac'], d['verified'], d['verified_last_step'])"
done
tail -2 gpurun_out/bench_err.log
