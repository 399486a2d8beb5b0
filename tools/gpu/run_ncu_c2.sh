# one ncu --set full capture of k_sort_fused (config $CFG, default c2) + per-line stall summary
CFG=${CFG:-c2}
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 120 python tools/prof_step.py --config $CFG --steps 3 > gpurun_out/prof_step.log 2>&1; rc=$?; echo step=$rc
if [ $rc -eq 0 ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${KERN:-k_sort_fused} -s ${SKIP:-2} -c 1 -f -o gpurun_out/full_$CFG \
  python tools/prof_step.py --config $CFG > gpurun_out/ncu_full_$CFG.log 2>&1; echo full=$?
python tools/ncu_summary.py gpurun_out/full_$CFG.ncu-rep > gpurun_out/full_${CFG}_summary.txt 2>&1
python tools/ncu_lines.py gpurun_out/full_$CFG.ncu-rep ${KERN:-k_sort_fused} 60 > gpurun_out/full_${CFG}_lines.txt 2>&1
cat gpurun_out/full_${CFG}_summary.txt
fi
