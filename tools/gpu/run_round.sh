# Round-end evidence: smoke + pytest -m gpu + all bench lines (run_all.sh), ncu launch list and
# full captures (run_prof.sh), phase stamps (libdialsort_phase.so, built before the call).
bash tools/gpu/run_all.sh
bash tools/gpu/run_prof.sh
rm -f gpurun_out/phase_times.txt
for c in c2 c3-zipf c3-sorted c4; do
  timeout 300 python tools/phase_times.py $c 2>&1 | grep -A1 "rep 3" >> gpurun_out/phase_times.txt
done
timeout 300 python tools/phase_radix.py > gpurun_out/phase_radix.txt 2>&1; echo phase_radix=$?
