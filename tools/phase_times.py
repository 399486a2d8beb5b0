"""Per-phase timing of the fused DialSort kernels in a back-to-back step loop (debug)."""
import os
import sys

os.environ["DIALSORT_PHASE_TIMING"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2605_16667_b200 as ds  # noqa: E402

cfgname = sys.argv[1] if len(sys.argv) > 1 else "c2"
cfg = bench.CONFIGS[cfgname]
dev = torch.device("cuda:0")
keys = [bench.make_device_input(cfg, 20260321, dev) for _ in range(5)]
outs = [torch.empty_like(k) for k in keys]
ctx = ds.Context(0, max_n=cfg["n"], max_U=cfg["U"])
names = ["ingest", "sync", "flush", "barrier1", "merge_scan", "offsets_issued", "rows_summed", "expand_start"]
for rep in range(3):
    ctx.debug_phase_ns()
    for i in range(1):  # one isolated step (previous work drained)
        ctx.sort(keys[rep % 5], cfg["U"], out=outs[rep % 5])
    torch.cuda.synchronize()
    t = ctx.debug_phase_ns()
    print(cfgname, "isolated step phase end times (us):", {n: round(v / 1e3, 2) for n, v in zip(names, t)})
