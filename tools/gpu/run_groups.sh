# batched-sort CTA groups: kFPassTiles 48 (variant p48) with 4/5/6 groups vs base
python -c "import __graft_entry__ as g; g.build()" >/dev/null
for c in c2 c3-zipf c3-sorted; do
for cfg in "base 4" "p48 4" "p48 5" "p48 6" "base 4" "p48 5" "p48 6"; do
  set -- $cfg
  vv=$1; [ "$1" = base ] && vv=
  DIALSORT_LIB_VARIANT=$vv DIALSORT_BATCH_GROUPS=$2 timeout 300 python bench.py --config $c --steps 320 --warmup 32 --no-cpu-baseline --no-e2e > gpurun_out/v.json 2>>gpurun_out/bench_err.log
  python -c "import json;d=json.load(open('gpurun_out/v.json'));print('[$1 L=$2] $c', '%.4f ms'%d['ms_per_step'], 'best %.4f'%d['reps']['best_ms_per_step'], 'frac %.3f'%d['roofline']['frac'], d['verified'], d['verified_last_step'])"
done; done
