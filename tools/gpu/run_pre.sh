TLIM=1500 bash tools/gpu/run_tests.sh
VARIANTS="base nohot base nohot" CONFIGS="c2 c3-zipf" BATCHES="32 1" bash tools/gpu/run_var_ab.sh
timeout 300 python tools/skew_scale.py 2>&1 | tail -4
timeout 300 python bench.py --config c4 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/c4.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/c4.json'));print('c4', d['ms_per_step'], d['roofline']['kernels_ms'], d['verified'])"
