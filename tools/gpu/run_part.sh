# hierarchical partition: parity tests + c4 sampled vs exact (and library variants in VARIANTS)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1200 python -m pytest tests/test_gpu.py tests/test_gpu_multi.py tests/test_gpu_next.py -m gpu -x -q -k "${KEXPR:-partition_modes or c4 or hierarch or universe or unaligned or in_place or key_range or loopback or graph}" > gpurun_out/pytest_part.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_part.log
for v in ${VARIANTS:-base}; do
  vv=$v; [ "$v" = base ] && vv=
  for m in ${MODES:-0 1}; do DIALSORT_LIB_VARIANT=$vv timeout 300 python bench.py --config c4 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --part-mode $m > gpurun_out/c4_$m.json 2>>gpurun_out/bench_err.log; python -c "import json;d=json.load(open('gpurun_out/c4_$m.json'));r=d['roofline'];print('[$v] c4 part_mode=$m', '%.4f ms'%d['ms_per_step'], r['kernel'], 'frac %.3f'%r['frac'], r.get('kernels_ms'))"; done
done
