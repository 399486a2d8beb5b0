"""Per-phase timing of the batched sort (debug, libdialsort_phase.so): 32 c2 steps in one
k_sort_batch launch; the stamps of each CTA are those of its group's last step.  Prints, per
group, the median duration of each phase of that step (us)."""
import os
import sys

os.environ["DIALSORT_PHASE_TIMING"] = "1"
os.environ.setdefault("DIALSORT_LIB_VARIANT", "phase")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2605_16667_b200 as ds  # noqa: E402

cfgname = sys.argv[1] if len(sys.argv) > 1 else "c2"
cfg = bench.CONFIGS[cfgname]
dev = torch.device("cuda:0")
B = 32
ins = [bench.make_device_input(cfg, 20260321 + (i % 4), dev) for i in range(B)]
outs = [torch.empty_like(ins[0]) for _ in range(B)]
ctx = ds.Context(0, max_n=cfg["n"], max_U=cfg["U"])
names = ["ingest", "sync", "flush", "barrier1", "offsets", "batch_staged", "merged", "end", "flags_ready",
         "proj_start", "m_reduced", "flush_loop", "r_rows", "r_synced", "m_scanned", "m_Pwritten"]
order = [0, 1, 11, 2, 3, 4, 5, 10, 14, 15, 6, 9, 7]
for rep in range(3):
    ctx.debug_phase_cta()
    ctx.sort_batch(ins, cfg["U"], outs)
    torch.cuda.synchronize()
    st = ctx.debug_phase_cta().astype(np.float64) / 1e3
    if rep == 0:
        continue
    G = len(st) // 4
    for g in range(4):
        rows = st[g * G:(g + 1) * G]
        prev = None
        parts = []
        for i in order:
            col = rows[:, 1 + i]
            if (col > 0).all():
                m = np.median(col)
                if prev is not None:
                    parts.append(f"{names[i]}+{m - prev:.2f}")
                else:
                    parts.append(f"{names[i]}@{m:.2f}")
                prev = m
        print(f"{cfgname} rep {rep} group {g}: " + "  ".join(parts), flush=True)
