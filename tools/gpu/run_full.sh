# full GPU parity suite + sanitizer-size smoke of every kernel family + batched A/B of groups
bash tools/gpu/run_tests.sh
timeout 300 python tools/sanitize_run.py > gpurun_out/sanitize_plain.log 2>&1; echo sanitize_plain=$?; tail -1 gpurun_out/sanitize_plain.log
GROUPS_="4 5 6" BATCHES="32" CONFIGS="c2 c3-zipf" bash tools/gpu/run_batch_ab.sh
