# Round profiles: launch list of the default bench command (after it exits 0 without ncu),
# one ncu --set full capture of the dominant kernel of c2 / c4 / c5 via tools/prof_step.py.
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 300 python bench.py --steps 2 --warmup 3 > gpurun_out/prof_bench_plain.jsonl 2>gpurun_out/prof_bench_plain.err; rc=$?; echo bench_plain=$rc
if [ $rc -eq 0 ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv \
    python bench.py --steps 2 --warmup 3 > gpurun_out/prof_bench_ncu.log 2>&1; echo ncu_launches=$?
fi
for c in c2 c4 c5; do
  timeout 120 python tools/prof_step.py --config $c --steps 3 > gpurun_out/prof_step_$c.log 2>&1; echo step_$c=$?
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sort_fused -s 2 -c 1 -f -o gpurun_out/full_c2 \
  python tools/prof_step.py --config c2 > gpurun_out/ncu_full_c2.log 2>&1; echo full_c2=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_part_scatter -s 1 -c 1 -f -o gpurun_out/full_c4 \
  python tools/prof_step.py --config c4 > gpurun_out/ncu_full_c4.log 2>&1; echo full_c4=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sort_fused -s 17 -c 1 -f -o gpurun_out/full_c4f \
  python tools/prof_step.py --config c4 > gpurun_out/ncu_full_c4f.log 2>&1; echo full_c4f=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_radix_pass -s 4 -c 1 -f -o gpurun_out/full_c5 \
  python tools/prof_step.py --config c5 > gpurun_out/ncu_full_c5.log 2>&1; echo full_c5=$?
