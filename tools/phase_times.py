"""Per-phase timing of the fused DialSort kernels (debug): one isolated step at a time,
per-CTA %globaltimer stamps, printed as min / median / max over CTAs per phase."""
import os
import sys

os.environ["DIALSORT_PHASE_TIMING"] = "1"
# the stamps exist only in the -DDIALSORT_PHASE_MARKS=1 build (tools/build_variant.sh phase)
os.environ.setdefault("DIALSORT_LIB_VARIANT", "phase")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2605_16667_b200 as ds  # noqa: E402

cfgname = sys.argv[1] if len(sys.argv) > 1 else "c2"
verbose = len(sys.argv) > 2
if cfgname in bench.CONFIGS:
    cfg = bench.CONFIGS[cfgname]
else:  # "n,U,dist" (a synth distribution)
    n_, U_, d_ = cfgname.split(",")
    cfg = dict(n=int(float(n_)), U=int(U_), dist=d_)
dev = torch.device("cuda:0")
if cfgname in bench.CONFIGS:
    keys = [bench.make_device_input(cfg, 20260321, dev) for _ in range(5)]
else:
    import synth
    keys = [torch.from_numpy(synth.make(cfg["dist"], cfg["n"], cfg["U"], 20260321 + i)).to(dev) for i in range(5)]
outs = [torch.empty_like(k) for k in keys]
ctx = ds.Context(0, max_n=cfg["n"], max_U=max(cfg["U"], 256))
fused = True
names = ["ingest", "sync", "flush", "barrier1", "offsets", "batch_staged", "merged", "end", "flags_ready",
         "proj_start", "m_reduced", "flush_loop", "r_rows", "tbl_built", "m_scanned", "m_Pwritten"]
for rep in range(4):
    ctx.debug_phase_cta()
    for _ in range(int(os.environ.get("PHASE_BACK_TO_BACK", "1"))):  # stamps: the last launch
        if cfg["dist"] == "int32":
            ctx.sort_int32(keys[rep % 5], out=outs[rep % 5])
        else:
            ctx.sort(keys[rep % 5], cfg["U"], out=outs[rep % 5])
    torch.cuda.synchronize()
    st = ctx.debug_phase_cta().astype(np.float64) / 1e3
    if rep == 0 or len(st) == 0:
        continue  # first call: warm-up
    print(f"{cfgname} rep {rep}: {len(st)} CTAs, phase time after the first CTA start (us) min/median/max:")
    cols = [("start", st[:, 0])] + [(n, st[:, 1 + i]) for i, n in enumerate(names)]
    print("   " + "  ".join(f"{n}={c[c > 0].min():.2f}/{np.median(c[c > 0]):.2f}/{c.max():.2f}"
                            for n, c in cols if n and (c > 0).any()))
    if verbose and fused:
        late = np.argsort(-st[:, 8])[:8]  # by end (phase 7)
        for b in late:
            print(f"   late CTA {b}: projection {st[b, 8] - st[b, 10]:.2f} us;",
                  " ".join(f"{n}={st[b, 1 + i]:.2f}" for i, n in enumerate(names) if n))
        pj = st[:, 8] - st[:, 10]
        print("   projection duration min/median/max %.2f/%.2f/%.2f us" % (pj.min(), np.median(pj), pj.max()))
