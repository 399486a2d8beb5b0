"""Run a few hot-path steps of one bench config (the command ncu profiles; no timing).
--batch B: B steps per dialsort_sort_batch_async call (the bench's batch mode)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2605_16667_b200 as ds  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--batch", type=int, default=1)
a = ap.parse_args()
cfg = bench.CONFIGS[a.config]
dev = torch.device("cuda:0")
keys = bench.make_device_input(cfg, 20260321, dev)
ctx = ds.Context(0, max_n=cfg["n"], max_U=max(cfg["U"], 256))
if a.batch > 1:
    ins = [keys] + [keys.clone() for _ in range(a.batch - 1)]
    outs = [torch.empty_like(keys) for _ in range(a.batch)]
    for _ in range(a.steps):
        ctx.sort_batch(ins, cfg["U"], outs)
else:
    out = torch.empty_like(keys)
    for _ in range(a.steps):
        if cfg["dist"] == "int32":
            ctx.sort_int32(keys, out=out)
        else:
            ctx.sort(keys, cfg["U"], out=out)
ctx.sync()
torch.cuda.synchronize()
print("ok", a.config, a.steps, a.batch)
