"""One rank's step of the multi-GPU path at G virtual ranks on ONE GPU (loopback communicators):
c2/8 (1.25e6 keys per rank, U = 65536) and c4/8 (1.25e8 keys per rank, U = 2^20).  Each step of
rank 0 is timed with CUDA events on its own (scatter: local histogram + stores into the owners'
slots + signal; gather: slot sum + total all-gather; project: offsets + slice projection); the
other ranks' steps run untimed in between so that every wait is already satisfied.  The step of a
real rank adds the exchange's wait for the slowest peer and NVLink latency (not measurable here)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2605_16667_b200 as ds  # noqa: E402
import synth  # noqa: E402

G = 8
dev = torch.device("cuda:0")
for name, n, U in [("c2/8", 10_000_000, 65536), ("c4/8", 1_000_000_000, 1 << 20)]:
    nl = n // G
    ctxs = [ds.Context(0, max_n=nl, max_U=U) for _ in range(G)]
    comms = [ds.Comm(ctxs[g], G, g, U, 0) for g in range(G)]
    for c in comms:
        c.connect_local(comms)
    shards = [synth.device_uniform(nl, U, lo=g * nl, device=dev) for g in range(G)]
    L = U // G
    out = torch.empty(2 * nl + (1 << 20), dtype=torch.int32, device=dev)
    cnt = torch.zeros(2, dtype=torch.int64, device=dev)
    times = {"scatter": [], "gather": [], "project": []}
    for it in range(6):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
        for g in range(G):
            if g == 0:
                ev[0].record()
            comms[g].scatter(shards[g], U)
            if g == 0:
                ev[1].record()
        for g in range(G):
            if g == 0:
                ev[2].record()
            comms[g].gather(U)  # (into the communicator's own slice buffer, which project(U, None) reads)
            if g == 0:
                ev[3].record()
        for g in range(G):
            o = out if g == 0 else torch.empty(2 * nl + (1 << 20), dtype=torch.int32, device=dev)
            cc = cnt if g == 0 else torch.zeros(2, dtype=torch.int64, device=dev)
            if g == 0:
                ev[4].record()
            comms[g].project(U, None, o, cc[0:1], cc[1:2])
            if g == 0:
                ev[5].record()
        torch.cuda.synchronize()
        for c in ctxs:
            c.sync()
        if it >= 1:
            times["scatter"].append(ev[0].elapsed_time(ev[1]))
            times["gather"].append(ev[2].elapsed_time(ev[3]))
            times["project"].append(ev[4].elapsed_time(ev[5]))
    # rank 0's output against the oracle's sharded reading (c2/8; c4/8: H slice only, sampled)
    ok = None
    if n <= 10_000_000:
        x = synth.uniform(n, U)
        Hr, outr, cr, offr = oracle.sharded_rank(x, U, G, 0)
        ok = bool(int(cnt[0]) == cr and int(cnt[1]) == offr and np.array_equal(out[:cr].cpu().numpy(), outr))
    med = {k: float(np.median(v)) for k, v in times.items()}
    step = sum(med.values())
    alg = 8 * nl + 8 * U + 8 * L  # per GPU 8n/G + 8U + 8U/G
    print(json.dumps({"config": name, "G": G, "keys_per_rank": nl, "U": U, "ms": med, "rank_step_ms": step,
                      "rank_keys_s": nl / (step * 1e-3), "alg_bytes": alg,
                      "frac_of_measured": alg / (step * 1e-3) / 1e9 / 6540.8, "verified_rank0": ok}), flush=True)
    del shards, ctxs, comms
    torch.cuda.empty_cache()
