"""Device time of single sorts at a given (n, U) (A/B helper): python tools/time_u.py n U [reps]."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import paper_2605_16667_b200 as ds  # noqa: E402
import oracle  # noqa: E402
import synth  # noqa: E402

n, U = int(sys.argv[1]), int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
dev = torch.device("cuda:0")
x = synth.uniform(n, U, seed=3)
k = torch.from_numpy(x).to(dev)
o = torch.empty_like(k)
ctx = ds.Context(0, max_n=n, max_U=U)
for _ in range(2):
    ctx.sort(k, U, out=o)
ctx.sync()
ok = bool(np.array_equal(o[:: max(1, n // 1000003)].cpu().numpy(), oracle.sort(x, U)[:: max(1, n // 1000003)]))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record()
for _ in range(reps):
    ctx.sort(k, U, out=o)
e1.record()
ctx.sync()
torch.cuda.synchronize()
print(f"n={n} U={U} {e0.elapsed_time(e1) / reps:.4f} ms/sort sampled_ok={ok} lib={os.environ.get('DIALSORT_LIB_VARIANT', '')} ring={os.environ.get('DIALSORT_PART_RING', '1')}")
