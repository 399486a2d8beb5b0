import os, sys
os.environ["DIALSORT_PHASE_TIMING"] = "1"
os.environ.setdefault("DIALSORT_LIB_VARIANT", "phase")
sys.path.insert(0, os.getcwd())
import numpy as np, torch, bench
import paper_2605_16667_b200 as ds
cfg = bench.CONFIGS["c2"]
dev = torch.device("cuda:0")
keys = bench.make_device_input(cfg, 20260321, dev); out = torch.empty_like(keys)
ctx = ds.Context(0, max_n=cfg["n"], max_U=cfg["U"])
for r in range(3):
    ctx.debug_phase_cta(); ctx.sort(keys, cfg["U"], out=out); torch.cuda.synchronize()
st = ctx.debug_phase_cta().astype(np.int64)
v = st[st > 0]
print("stamp values mod 32:", np.bincount(v % 32)[:32].nonzero()[0][:10], " mod 1000 sample:", (v % 1000)[:20])
print("CTA 0:", st[0])
