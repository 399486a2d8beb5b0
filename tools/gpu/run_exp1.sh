python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
VARIANTS="noclaim base" MODES="0" KEXPR="partition_modes and 1048576 and 0" bash tools/gpu/run_part.sh
for k in default 16384 8192 4096; do
  if [ $k = default ]; then timeout 300 python tools/kpc_ab.py; else DIALSORT_FUSED_KPC=$k timeout 300 python tools/kpc_ab.py; fi
done 2>&1 | grep -v Warn
