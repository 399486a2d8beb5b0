# Round-2 (session 2) evidence after the ring placement: default bench line, all-config lines,
# c4 exact schedule, per-rank loopback timing, launch list of the default bench, ncu --set full of
# the ring placement.
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 600 python bench.py > gpurun_out/r02s2_bench_default.jsonl 2> gpurun_out/r02s2_bench_default.err; echo bench=$?
rm -f gpurun_out/r02s2_bench_all.jsonl
for c in c2 c3-zipf c3-sorted c3-reverse c3-hot1 c1 c5 c4 c4-wide; do
  timeout 300 python bench.py --config $c --steps 256 --warmup 32 --no-cpu-baseline --no-e2e >> gpurun_out/r02s2_bench_all.jsonl 2>> gpurun_out/r02s2_bench_all.err
done
timeout 300 python bench.py --config c4 --part-mode 1 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02s2_bench_c4_exact.jsonl 2>>gpurun_out/r02s2_bench_all.err
DIALSORT_PART_RING=0 timeout 300 python bench.py --config c4 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02s2_bench_c4_subtile.jsonl 2>>gpurun_out/r02s2_bench_all.err
timeout 300 python tools/rank_step.py > gpurun_out/r02s2_rank_step.jsonl 2> gpurun_out/r02s2_rank_step.err; echo rank_step=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02s2_launches_bench.csv \
  python bench.py --steps 64 --warmup 32 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1; echo ncu_launches=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_part_place_ring -s 1 -c 1 -f -o gpurun_out/r02s2_full_c4_ring \
  python tools/prof_step.py --config c4 --steps 3 > gpurun_out/ncu_full_c4_ring.log 2>&1; echo full_c4_ring=$?
python tools/ncu_summary.py gpurun_out/r02s2_full_c4_ring.ncu-rep > gpurun_out/r02s2_ncu_c4_k_part_place_ring_summary.txt 2>&1
python tools/ncu_sass_hot.py gpurun_out/r02s2_full_c4_ring.ncu-rep k_part_place_ring 40 > gpurun_out/r02s2_ncu_c4_k_part_place_ring_hot.txt 2>&1
rm -f gpurun_out/r02s2_full_c4_ring.ncu-rep
du -sh gpurun_out
