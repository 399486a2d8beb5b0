"""Small invocations of every kernel family, for compute-sanitizer (memcheck / racecheck /
synccheck): sorts on every universe path, radix (both pass variants), queries, coded domains,
the batched sort and the multi-GPU exchange (G = 2 virtual ranks).  n <= 1e5."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2605_16667_b200 as ds  # noqa: E402
import synth  # noqa: E402

dev = torch.device("cuda:0")
c = ds.Context(0, max_n=100_000, max_U=1 << 20)
ok = True


def chk(name, got, ref):
    global ok
    good = np.array_equal(got, ref)
    ok &= good
    print(f"{name}: {'ok' if good else 'MISMATCH'}", flush=True)


for U, n in [(256, 100_000), (65536, 100_000), (20000, 60_000), (1 << 20, 100_000), ((1 << 22) + 7, 50_000)]:
    x = synth.uniform(n, U, seed=U)
    out = c.sort(torch.from_numpy(x).to(dev), U)
    c.sync()
    chk(f"sort U={U}", out.cpu().numpy(), oracle.sort(x, U))
x = np.full(100_000, 5, dtype=np.int32)
out = c.sort(torch.from_numpy(x).to(dev), 65536)  # packed-counter overflow fallback
c.sync()
chk("sort all-equal (overflow)", out.cpu().numpy(), x)
x = synth.zipf(100_000, 65536, seed=1)
out = c.sort(torch.from_numpy(x).to(dev), 65536)
c.sync()
chk("sort zipf (share mode)", out.cpu().numpy(), oracle.sort(x, 65536))
for v in (3, 4):
    c.set_option(ds._lib.OPT_RADIX_VARIANT, v)
    x = synth.full_int32(100_000, seed=v)
    y = c.sort_int32(torch.from_numpy(x).to(dev))
    c.sync()
    chk(f"radix pass{v}", y.cpu().numpy(), oracle.radix_sort_i32(x))
H = c.histogram(torch.from_numpy(synth.uniform(50_000, 4096)).to(dev), 4096)
q = c.query(H, ds._lib.Q_RANGE_COUNT, torch.tensor([[0, 4095], [10, 20]], dtype=torch.int32, device=dev))
D, cnt, iso = c.support_set(H)
f = c.query(H, ds._lib.Q_FREQUENCY, torch.arange(100, dtype=torch.int32, device=dev))
c.sync()
chk("queries", np.array([int(q[0])]), np.array([50_000]))
items = torch.randint(0, 200, (77_777,), dtype=torch.uint8, device=dev)
dec = torch.arange(256, dtype=torch.int32, device=dev) * 2
o = c.sort_domain(items, 256, decode=dec)
c.sync()
chk("domain u8", o.cpu().numpy(), oracle.sort_domain(items.cpu().numpy(), 256, decode=dec.cpu().numpy()))
xs = [synth.uniform(90_000 + j, 65536, seed=j) for j in range(4)]
outs = c.sort_batch([torch.from_numpy(x).to(dev) for x in xs], 65536)
c.sync()
chk("batch", np.concatenate([o.cpu().numpy() for o in outs]), np.concatenate([oracle.sort(x, 65536) for x in xs]))
ctxs = [ds.Context(0) for _ in range(2)]
comms = [ds.Comm(ctxs[g], 2, g, 65536, 100_000) for g in range(2)]
for cm in comms:
    cm.connect_local(comms)
x = synth.uniform(100_000, 65536, seed=9)
sh = [torch.from_numpy(x[g * 50_000:(g + 1) * 50_000].copy()).to(dev) for g in range(2)]
outs = [torch.empty(100_000, dtype=torch.int32, device=dev) for _ in range(2)]
cnts = [torch.zeros(2, dtype=torch.int64, device=dev) for _ in range(2)]
for g in range(2):
    comms[g].scatter(sh[g], 65536)
for g in range(2):
    comms[g].gather(65536)
for g in range(2):
    comms[g].project(65536, None, outs[g], cnts[g][0:1], cnts[g][1:2])
for cx in ctxs:
    cx.sync()
chk("sharded G=2", np.concatenate([outs[g][:int(cnts[g][0])].cpu().numpy() for g in range(2)]), oracle.sort(x, 65536))
xr = synth.full_int32(100_000, seed=3)
shr = [torch.from_numpy(xr[g * 50_000:(g + 1) * 50_000].copy()).to(dev) for g in range(2)]
for g in range(2):
    comms[g].radix_hist(shr[g])
for g in range(2):
    comms[g].radix_split(shr[g], 100_000, cnts[g][0:1], cnts[g][1:2])
for g in range(2):
    comms[g].radix_local(outs[g])
for cx in ctxs:
    cx.sync()
chk("sharded radix G=2", np.concatenate([outs[g][:int(cnts[g][0])].cpu().numpy() for g in range(2)]),
    oracle.radix_sort_i32(xr))
print("ALL OK" if ok else "FAILURES")
sys.exit(0 if ok else 1)
