# CUDA-graph capture debugging + the graph test + library A/B (bounded)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 180 python tools/graph_debug.py 2>&1 | tail -20
timeout 400 python -m pytest tests/test_gpu_next.py -q -x -m gpu -k "graph" 2>&1 | tail -5
VARIANTS="head base head base" CONFIGS=c2 BATCHES="32 1" bash tools/gpu/run_var_ab.sh
