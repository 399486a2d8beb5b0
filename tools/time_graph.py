"""Device time of one sort at (n, U) replayed from a CUDA graph (no host overhead; A/B helper):
python tools/time_graph.py n U [dist]."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import paper_2605_16667_b200 as ds  # noqa: E402
import oracle  # noqa: E402
import synth  # noqa: E402

n, U = int(sys.argv[1]), int(sys.argv[2])
dist = sys.argv[3] if len(sys.argv) > 3 else "uniform"
dev = torch.device("cuda:0")
x = synth.make(dist, n, U, 7)
k = torch.from_numpy(x).to(dev)
outs = [torch.empty_like(k) for _ in range(2)]
ctx = ds.Context(0, max_n=n, max_U=U)
s = torch.cuda.Stream(dev)
with torch.cuda.stream(s):
    for o in outs:
        ctx.sort(k, U, out=o)
    ctx.sync()
    g = torch.cuda.CUDAGraph()
    steps = 32
    with torch.cuda.graph(g, stream=s):
        for i in range(steps):
            ctx.sort(k, U, out=outs[i % 2])
    for _ in range(2):
        g.replay()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        g.replay()
        e1.record(s)
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / steps)
ok = bool(np.array_equal(outs[1].cpu().numpy(), oracle.sort(x, U)))
print(f"n={n} U={U} {dist} {best * 1000:.2f} us/sort (graph) ok={ok} lib={os.environ.get('DIALSORT_LIB_VARIANT', '')}")
