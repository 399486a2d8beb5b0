# Round-2 evidence: default bench line, all-config lines, paper grid, per-rank loopback timing,
# launch list, ncu --set full captures of the dominant kernels, phase stamps.
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
bash tools/build_variant.sh phase > /dev/null 2>&1; echo phase_lib=$?
timeout 600 python bench.py > gpurun_out/r02_bench_default.jsonl 2> gpurun_out/r02_bench_default.err; echo bench=$?
rm -f gpurun_out/r02_bench_all.jsonl
for c in c2 c3-zipf c3-sorted c3-reverse c3-hot1 c1 c5 c4 c4-wide; do
  timeout 300 python bench.py --config $c --steps 256 --warmup 32 --no-cpu-baseline --no-e2e >> gpurun_out/r02_bench_all.jsonl 2>> gpurun_out/r02_bench_all.err
done
timeout 300 python bench.py --config c4 --part-mode 1 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02_bench_c4_exact.jsonl 2>>gpurun_out/r02_bench_all.err
timeout 300 python bench.py --config c2 --batch 1 --steps 300 --warmup 10 --no-cpu-baseline --no-e2e > gpurun_out/r02_bench_c2_single.jsonl 2>>gpurun_out/r02_bench_all.err
timeout 900 python bench.py --grid > gpurun_out/r02_paper_grid.jsonl 2> gpurun_out/r02_paper_grid.err; echo grid=$?
timeout 300 python tools/rank_step.py > gpurun_out/r02_rank_step.jsonl 2> gpurun_out/r02_rank_step.err; echo rank_step=$?
timeout 120 python tools/phase_times.py c2 > gpurun_out/r02_phase_c2.txt 2>&1; echo phase=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_bench.csv \
  python bench.py --steps 64 --warmup 32 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1; echo ncu_launches=$?
for spec in "c2 k_sort_batch 32 1" "c2 k_sort_fused 1 2" "c3-zipf k_sort_fused 1 2" "c3-sorted k_sort_fused 1 2" "c5 k_radix_pass 1 4" "c4 k_part_place 1 2" "c4 k_sort_batch 1 1"; do
  set -- $spec
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$2 -s $4 -c 1 -f -o gpurun_out/r02_full_${1}_$2 \
    python tools/prof_step.py --config $1 --batch $3 --steps 3 > gpurun_out/ncu_full_${1}_$2.log 2>&1; echo full_$1_$2=$?
  python tools/ncu_summary.py gpurun_out/r02_full_${1}_$2.ncu-rep > gpurun_out/r02_ncu_${1}_$2_summary.txt 2>&1
  python tools/ncu_sass_hot.py gpurun_out/r02_full_${1}_$2.ncu-rep $2 40 > gpurun_out/r02_ncu_${1}_$2_hot.txt 2>&1
  rm -f gpurun_out/r02_full_${1}_$2.ncu-rep  # (gpurun copies back at most 64 MiB)
done
du -sh gpurun_out
