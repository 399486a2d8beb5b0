# one ncu --set full capture of k_radix_pass (c5) + summary + per-SASS dump
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 120 python tools/prof_step.py --config c5 --steps 3 > gpurun_out/prof_step_c5.log 2>&1; rc=$?; echo step_c5=$rc
if [ $rc -eq 0 ]; then
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_radix_pass -s 4 -c 1 -f -o gpurun_out/full_c5 \
  python tools/prof_step.py --config c5 > gpurun_out/ncu_full_c5.log 2>&1; echo full_c5=$?
python tools/ncu_summary.py gpurun_out/full_c5.ncu-rep > gpurun_out/full_c5_summary.txt 2>&1
fi
