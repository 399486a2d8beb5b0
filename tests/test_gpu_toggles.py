"""GPU parity of the library's design / debug switches (environment variables read once per
process, so each case runs in a subprocess): every alternative schedule they select must give
the oracle's H and output bit for bit.

  DIALSORT_PART_RING=0     sub-tile placement instead of the ring placement (U <= 2^20)
  DIALSORT_PART_WIDE=1     the wide (per-CTA counter) partition for U <= 2^22
  DIALSORT_HIER_BATCH=0    one launch per universe block instead of the batched block steps
  DIALSORT_NO_HIER=1       the L2 path (global H, k_scan + k_expand) for U > 98304
  DIALSORT_FUSED_KPC=...   the fused step's grid sized for other keys-per-CTA counts
  DIALSORT_BATCH_GROUPS=2  the batched sort on 2 CTA groups
  DIALSORT_NO_FIFO=1       no FIFO between co-resident launches (single stream)
  DIALSORT_NO_PDL=1        launches without programmatic dependent launch
  DIALSORT_SMALL=0         small inputs on the fused co-resident grid instead of one cluster
"""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys
sys.path.insert(0, %(root)r)
import numpy as np, torch
import oracle, synth
import paper_2605_16667_b200 as ds
dev = torch.device("cuda:0")
c = ds.Context(0, max_n=3_000_000, max_U=1 << 22)
cases = [(3_000_001, 1 << 20, "uniform"), (2_000_003, 1 << 20, "zipf"), (1_000_000, (1 << 22) - 3, "uniform"),
         (1_000_001, 65536, "uniform"), (999_999, 300_000, "sorted"), (70_000, 1 << 20, "uniform"),
         (100_000, 256, "uniform"), (99_999, 8192, "zipf"), (5_001, 1000, "sorted")]
for n, U, dist in cases:
    x = synth.make(dist, n, U, 11)
    k = torch.from_numpy(x).to(dev)
    H = torch.empty(U, dtype=torch.int32, device=dev)
    o = c.sort(k, U, H=H)
    c.sync()
    Hr = oracle.histogram(x, U)
    assert np.array_equal(H.cpu().numpy().view(np.uint32).astype(np.uint64), Hr), ("H", n, U, dist)
    assert np.array_equal(o.cpu().numpy(), oracle.project(Hr)), ("out", n, U, dist)
xs = [synth.uniform(400_000 + 13 * j, 65536, seed=j) for j in range(5)]
outs = c.sort_batch([torch.from_numpy(v).to(dev) for v in xs], 65536)
c.sync()
for v, o in zip(xs, outs):
    assert np.array_equal(o.cpu().numpy(), oracle.sort(v, 65536)), "batch"
y = synth.full_int32(1_000_003)
assert np.array_equal(c.sort_int32(torch.from_numpy(y).to(dev)).cpu().numpy(), oracle.radix_sort_i32(y)), "radix"
print("ok")
"""


@pytest.mark.parametrize("env", [
    {"DIALSORT_PART_RING": "0"},
    {"DIALSORT_PART_WIDE": "1"},
    {"DIALSORT_HIER_BATCH": "0"},
    {"DIALSORT_NO_HIER": "1"},
    {"DIALSORT_FUSED_KPC": "32768"},
    {"DIALSORT_BATCH_GROUPS": "2"},
    {"DIALSORT_NO_FIFO": "1", "DIALSORT_NO_PDL": "1"},
    {"DIALSORT_SMALL": "0"},
], ids=lambda e: ",".join(f"{k}={v}" for k, v in e.items()))
def test_switch_parity(cuda_dev, env):
    r = subprocess.run([sys.executable, "-c", SCRIPT % {"root": ROOT}], env={**os.environ, **env},
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), (r.stdout[-2000:], r.stderr[-4000:])
