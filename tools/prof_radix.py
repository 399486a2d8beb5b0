"""A few radix sorts at c5 size (for ncu)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
import paper_2605_16667_b200 as ds
n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
x = synth.device_full_int32(n, device="cuda:0")
y = torch.empty_like(x)
ctx = ds.Context(0, max_n=n)
for _ in range(2):
    ctx.sort_int32(x, out=y)
ctx.sync()
print("ok")
