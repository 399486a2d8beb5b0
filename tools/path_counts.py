"""Debug (libdialsort_pathcnt.so, -DDIALSORT_EXP_PATHCNT=1): per-CTA projection duration vs the
number of super-blocks that took each projection path (none / distinct / marks)."""
import os
import sys
os.environ["DIALSORT_PHASE_TIMING"] = "1"
os.environ.setdefault("DIALSORT_LIB_VARIANT", "pathcnt")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import bench  # noqa: E402
import paper_2605_16667_b200 as ds  # noqa: E402

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3-zipf"]
keys = bench.make_device_input(cfg, 20260321, torch.device("cuda:0"))
out = torch.empty_like(keys)
ctx = ds.Context(0, max_n=cfg["n"], max_U=cfg["U"])
for _ in range(3):
    ctx.debug_phase_cta()
    ctx.sort(keys, cfg["U"], out=out)
    torch.cuda.synchronize()
raw = ctx.debug_phase_cta()
st = raw.astype(np.float64)
pj = (st[:, 8] - st[:, 10]) / 1e3   # end - projection start (us)
cnt = (raw[:, 12:15].astype(np.int64) - raw[:, 15:16].astype(np.int64))  # t + count minus t
order = np.argsort(-pj)
print("CTA  proj_us  none distinct marks")
for b in list(order[:10]) + list(order[-5:]):
    print(f"{b:4d} {pj[b]:7.2f} {cnt[b, 0]:5d} {cnt[b, 1]:8d} {cnt[b, 2]:5d}")
