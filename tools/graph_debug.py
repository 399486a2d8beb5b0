"""Capture each public call alone into a CUDA graph and replay it twice (bounded; debugging aid)."""
import sys
sys.path.insert(0, '/root/repo')
import torch, numpy as np
import paper_2605_16667_b200 as ds, synth, oracle
dev = torch.device('cuda:0')
c = ds.Context(0, max_n=200000, max_U=65536)
U = 4096
x = torch.from_numpy(synth.uniform(100000, U)).to(dev)
xb = [torch.from_numpy(synth.uniform(90000 + j, U, seed=j)).to(dev) for j in range(3)]
xr = torch.from_numpy(synth.full_int32(50000)).to(dev)
H = torch.empty(U, dtype=torch.int32, device=dev)
o = torch.empty_like(x)
ob = [torch.empty_like(t) for t in xb]
orr = torch.empty_like(xr)
q = torch.arange(0, U, 7, dtype=torch.int32, device=dev)
ops = {
    "sort": lambda: c.sort(x, U, out=o, H=H),
    "sort_batch": lambda: c.sort_batch(xb, U, ob),
    "reconstruct": lambda: c.reconstruct(H, o),
    "sort_int32": lambda: c.sort_int32(xr, out=orr),
    "query": lambda: c.query(H, ds._lib.Q_FREQUENCY, q),
}
for name, f in ops.items():
    f(); c.sync(); torch.cuda.synchronize()
    try:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            f()
        for _ in range(2):
            g.replay()
        torch.cuda.synchronize(); c.sync()
        print(name, "ok", flush=True)
    except Exception as e:
        print(name, "FAIL", str(e)[:300], flush=True)
        try:
            torch.cuda.synchronize()
        except Exception as e2:
            print("  sync after:", str(e2)[:200]); break
