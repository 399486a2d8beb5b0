# ncu --set full of k_part_scatter_est (c4, sampled partition) + hot SASS; phase stamps of c1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 120 python tools/prof_step.py --config c4 --steps 3 > gpurun_out/prof_step_c4.log 2>&1; rc=$?; echo step_c4=$rc
if [ $rc -eq 0 ]; then
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_part_scatter_est -s 1 -c 1 -f -o gpurun_out/full_c4est \
  python tools/prof_step.py --config c4 > gpurun_out/ncu_full_c4est.log 2>&1; echo full_c4est=$?
python tools/ncu_summary.py gpurun_out/full_c4est.ncu-rep > gpurun_out/full_c4est_summary.txt 2>&1
python tools/ncu_sass_hot.py gpurun_out/full_c4est.ncu-rep k_part_scatter_est 70 > gpurun_out/full_c4est_hot.txt 2>&1
cat gpurun_out/full_c4est_summary.txt
fi
timeout 120 python tools/phase_times.py c1 > gpurun_out/phase_c1.txt 2>&1; echo phase=$?; cat gpurun_out/phase_c1.txt | head -20
