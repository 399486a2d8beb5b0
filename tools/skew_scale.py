"""Single-call time of large skewed sorts (where the packed 16-bit counters can overflow per CTA:
n / C > 65535 and a key's share p > 65535 C / n): uniform vs Zipf(1.2) vs one hot key."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import paper_2605_16667_b200 as ds  # noqa: E402
import synth  # noqa: E402
import oracle  # noqa: E402

dev = torch.device("cuda:0")
for n, U in ((10_000_000, 65536), (30_000_000, 65536), (100_000_000, 65536), (100_000_000, 1 << 20)):
    ctx = ds.Context(0, max_n=n, max_U=U)
    for dist in ("uniform", "zipf", "hot10"):
        if dist == "hot10":
            x = synth.uniform(n, U, seed=5)
            x[np.random.default_rng(5).random(n) < 0.10] = 4242 % U
        else:
            x = synth.make(dist, n, U, 20260321)
        k = torch.from_numpy(x).to(dev)
        o = torch.empty_like(k)
        for _ in range(3):
            ctx.sort(k, U, out=o)
        ctx.sync()
        ok = bool(np.array_equal(o.cpu().numpy(), oracle.sort(x, U)))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(10):
            ctx.sort(k, U, out=o)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        print(f"n={n} U={U} {dist}: {ms*1e3:.1f} us  {n / (ms * 1e-3) / 1e9:.1f} Gkeys/s ok={ok}", flush=True)
    del ctx
