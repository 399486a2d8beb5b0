import os, sys
os.environ["DIALSORT_PHASE_TIMING"] = "1"
sys.path.insert(0, "/root/repo")
import numpy as np, torch, bench, paper_2605_16667_b200 as ds
cfg = bench.CONFIGS["c3-zipf"]
dev = torch.device("cuda:0")
keys = bench.make_device_input(cfg, 20260321, dev)
out = torch.empty_like(keys)
H = torch.empty(cfg["U"], dtype=torch.int32, device=dev)
ctx = ds.Context(0, max_n=cfg["n"], max_U=cfg["U"])
for rep in range(3):
    ctx.debug_phase_cta()
    ctx.sort(keys, cfg["U"], out=out, H=H)
    torch.cuda.synchronize()
    st = ctx.debug_phase_cta().astype(np.float64) / 1e3
h = H.cpu().numpy().astype(np.int64)
T16 = 128
tiles = h.reshape(-1, T16).sum(1)
toff = np.concatenate([[0], np.cumsum(tiles)])
C = len(st); ntiles = len(tiles)
alpha = 2 * C * 16
cs = np.arange(ntiles + 1) * alpha + toff
T = cs[-1]
ps = st[:, 1 + 13]; en = st[:, 1 + 7]
order = np.argsort(-(en - ps))[:12]
for b in order:
    r0, r1 = T * b // C, T * (b + 1) // C
    ta = np.searchsorted(cs, r0, side="right") - 1; tb = np.searchsorted(cs, r1 - 1, side="right") - 1
    # positions of the slice and nonzero bins (starts) in them
    pos = 0; nz = 0
    for t in range(ta, tb + 1):
        s0 = cs[t] + alpha; e = cs[t + 1]
        lo, hi = max(r0, s0), min(r1, e)
        if lo < hi:
            pos += hi - lo
            nz += int((h[t*T16:(t+1)*T16] > 0).sum())
    print(f"CTA {b:3d}: proj {en[b]-ps[b]:6.2f} us  tiles {tb-ta+1:3d}  positions {pos:7d}  bins>0 in slice tiles {nz}")
