"""Stall samples and executed warp-instructions per CUDA source line of one kernel, from the
interleaved cuda,sass source page of an ncu report (needs -lineinfo).  Usage:
  python tools/ncu_lines.py report.ncu-rep <kernel regex> [top]"""
import csv
import subprocess
import sys
from collections import defaultdict

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", "regex:" + kern,
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
agg = defaultdict(lambda: [0, 0, ""])
fname, line, src = None, None, ""
seen_fn = set()
for r in csv.reader(raw.splitlines()):
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) == 2 and r[0] == "Function Name":
        if r[1] in seen_fn and len(seen_fn) > 0 and fname is None:
            break
        seen_fn.add(r[1])
        continue
    if len(r) < 8 or r[0] == "Line No":
        continue
    if r[0]:
        line, src = r[0], r[1]
        continue
    try:
        smp, ex = int(r[4] or 0), int(r[7] or 0)
    except ValueError:
        continue
    a = agg[(fname, line)]
    a[0] += smp
    a[1] += ex
    a[2] = src
tot = sum(v[0] for v in agg.values()) or 1
print(f"total stall samples {tot}")
for (f, ln), (smp, ex, s) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{100.0 * smp / tot:5.1f}% {ex:10d} {f}:{ln:5s} {s.strip()[:90]}")

# per-file-region totals (instructions executed, stall samples)
if len(sys.argv) > 4:
    reg = defaultdict(lambda: [0, 0])
    for (f, ln), (smp, ex, s) in agg.items():
        key = f
        for spec in sys.argv[4].split(";"):  # "file:lo-hi=name"
            fn, rest = spec.split(":")
            rng, name = rest.split("=")
            lo, hi = map(int, rng.split("-"))
            if f == fn and ln and ln.isdigit() and lo <= int(ln) <= hi:
                key = name
        reg[key][0] += smp
        reg[key][1] += ex
    totx = sum(v[1] for v in reg.values()) or 1
    for k, (smp, ex) in sorted(reg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k:28s} instr {ex:10d} ({100.0 * ex / totx:5.1f}%)  stall samples {100.0 * smp / tot:5.1f}%")
