"""A/B of the fused kernel's grid sizing (DIALSORT_FUSED_KPC keys per CTA): single-call device
time per sort, best of 7 blocks, for small and mid-size n (one line per config)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import numpy as np  # noqa: E402
import paper_2605_16667_b200 as ds  # noqa: E402
import synth  # noqa: E402
import oracle  # noqa: E402

dev = torch.device("cuda:0")
ctx = ds.Context(0, max_n=4_000_000, max_U=65536)
kpc = os.environ.get("DIALSORT_FUSED_KPC", "default")
for n in (10_000, 100_000, 300_000, 1_000_000, 3_000_000):
    for U in (256, 1024, 65536):
        for dist in ("uniform", "skewed"):
            x = synth.make(dist, n, U, 20260321)
            R = 8
            ins = [torch.from_numpy(x).to(dev) for _ in range(R)]
            outs = [torch.empty_like(ins[0]) for _ in range(R)]
            for i in range(5):
                ctx.sort(ins[i % R], U, out=outs[i % R])
            ctx.sync()
            ok = bool(np.array_equal(outs[4 % R].cpu().numpy(), oracle.sort(x, U)))
            kb = 100
            blk = []
            for r in range(7):
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for i in range(kb):
                    ctx.sort(ins[i % R], U, out=outs[i % R])
                e1.record()
                torch.cuda.synchronize()
                blk.append(e0.elapsed_time(e1) / kb * 1e3)
            ctx.sync()
            print(f"kpc={kpc} n={n} U={U} {dist}: best {min(blk):.2f} us median {sorted(blk)[3]:.2f} ok={ok}", flush=True)
