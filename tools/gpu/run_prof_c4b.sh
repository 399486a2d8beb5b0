# ncu --set full of c4's placement (k_part_place<true>) and block steps (k_sort_batch), + hot SASS
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 120 python tools/prof_step.py --config c4 --steps 3 > gpurun_out/prof_step_c4.log 2>&1; rc=$?; echo step_c4=$rc
if [ $rc -eq 0 ]; then
for kn in k_part_place k_sort_batch; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$kn -s 2 -c 1 -f -o gpurun_out/full_c4_$kn \
  python tools/prof_step.py --config c4 > gpurun_out/ncu_full_c4_$kn.log 2>&1; echo full_$kn=$?
python tools/ncu_summary.py gpurun_out/full_c4_$kn.ncu-rep > gpurun_out/full_c4_${kn}_summary.txt 2>&1
python tools/ncu_sass_hot.py gpurun_out/full_c4_$kn.ncu-rep $kn 60 > gpurun_out/full_c4_${kn}_hot.txt 2>&1
cat gpurun_out/full_c4_${kn}_summary.txt
done
fi
