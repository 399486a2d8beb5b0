"""Phase timing of one radix pass kernel sequence (debug)."""
import os, sys
os.environ["DIALSORT_PHASE_TIMING"] = "1"
os.environ.setdefault("DIALSORT_LIB_VARIANT", "phase")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
import paper_2605_16667_b200 as ds
n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
x = synth.device_full_int32(n, device="cuda:0")
y = torch.empty_like(x)
ctx = ds.Context(0, max_n=n)
ctx.sort_int32(x, out=y); torch.cuda.synchronize()
for _ in range(2):
    ctx.debug_phase_ns()
    ctx.sort_int32(x, out=y)
    torch.cuda.synchronize()
    t = ctx.debug_phase_ns()  # max over the 4 passes of (phase end - first start): cumulative
    print({k: round(v / 1e3, 1) for k, v in zip(["count", "bar1", "colscan", "bar2", "scatter"], t[:5])})
