"""Experiment: c2 sorts on L lanes (contexts capped at nsm/L CTAs, one stream each, batches
alternating) vs one full-grid context.  DIALSORT_NO_FIFO=1 must be set (lets the lanes overlap)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench, paper_2605_16667_b200 as ds, oracle
cfgname = sys.argv[1] if len(sys.argv) > 1 else "c2"
cfg = bench.CONFIGS[cfgname]
n, U = cfg["n"], cfg["U"]
dev = torch.device("cuda:0")
R = 8
ins = [bench.make_device_input(cfg, 20260321 + i, dev) for i in range(R)]
outs = [torch.empty_like(ins[0]) for _ in range(R)]
K = 400
for L in (1, 2, 3, 4):
    ctxs = [ds.Context(0, max_n=n, max_U=U) for _ in range(L)]
    for c in ctxs:
        c.set_option(ds._lib.OPT_MAX_CTAS, 148 // L)
    sts = [torch.cuda.Stream(dev) for _ in range(L)]
    def run(k0, k):
        for i in range(k0, k0 + k):
            with torch.cuda.stream(sts[i % L]):
                ctxs[i % L].sort(ins[i % R], U, out=outs[i % R])
    run(0, 20)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    cur = torch.cuda.current_stream(dev)
    e0.record(cur)
    for s in sts:
        s.wait_stream(cur)
    run(0, K)
    for s in sts:
        cur.wait_stream(s)
    e1.record(cur)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / K
    for i, c in enumerate(ctxs):
        with torch.cuda.stream(sts[i]):
            c.sync()
    ok = all(np.array_equal(outs[i].cpu().numpy(), oracle.sort(ins[i].cpu().numpy(), U)) for i in range(2))
    print(f"{cfgname} lanes={L} ctas/lane={148 // L}: {ms * 1e3:.2f} us per batch, {n / ms / 1e6:.3e} keys/s, verified={ok}", flush=True)
