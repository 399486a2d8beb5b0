# one ncu --set full capture of k_part_scatter (c4) + per-SASS hot spots
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 120 python tools/prof_step.py --config c4 --steps 3 > gpurun_out/prof_step_c4.log 2>&1; rc=$?; echo step_c4=$rc
if [ $rc -eq 0 ]; then
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_part_scatter -s 1 -c 1 -f -o gpurun_out/full_c4 \
  python tools/prof_step.py --config c4 > gpurun_out/ncu_full_c4.log 2>&1; echo full_c4=$?
python tools/ncu_summary.py gpurun_out/full_c4.ncu-rep > gpurun_out/full_c4_summary.txt 2>&1
python tools/ncu_sass_hot.py gpurun_out/full_c4.ncu-rep k_part_scatter 70 > gpurun_out/full_c4_hot.txt 2>&1
fi
