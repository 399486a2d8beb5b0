# batched-sort A/B: groups x batch size (x stagger), c2 and zipf
for c in ${CONFIGS:-c2 c3-zipf}; do
  for L in ${GROUPS_:-3 4}; do
    for B in ${BATCHES:-32 64}; do
      for ns in ${NOSTAG:-0}; do
      if [ $ns = 1 ]; then export DIALSORT_BATCH_NOSTAGGER=1; else unset DIALSORT_BATCH_NOSTAGGER; fi
      DIALSORT_BATCH_GROUPS=$L timeout 300 python bench.py --config $c --steps 640 --warmup 64 --batch $B --no-cpu-baseline --no-e2e > gpurun_out/bab.json 2>>gpurun_out/bench_err.log
      python -c "import json;d=json.load(open('gpurun_out/bab.json'));r=d['roofline'];print('$c L=$L B=$B nostag=$ns', '%.4f ms'%d['ms_per_step'], 'frac %.3f'%r['frac'], r['kernel'], 'single %.4f'%d['single_call']['ms_per_step'], 'best %.4f'%d['reps']['best_ms_per_step'], 'cv %.3f'%d['reps']['cv'], 'ok', d['verified'], d['verified_last_step'])"
      done
    done
  done
done
tail -3 gpurun_out/bench_err.log
