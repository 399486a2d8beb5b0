"""Per-SASS-instruction execution counts and stall samples of one kernel in an ncu report."""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 60
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", "regex:" + kern,
                      "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr = rows[1]
ia, isrc, iex, ismp = hdr.index("Address"), hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
body = []
for r in rows[2:]:  # first kernel instance only
    if r and r[0] == "Kernel Name":
        break
    if len(r) == len(hdr) and r[iex].isdigit():
        body.append(r)
tot = sum(int(r[iex] or 0) for r in body)
tots = sum(int(r[ismp] or 0) for r in body)
print(f"total warp-instructions {tot}, stall samples {tots}")
for n, r in enumerate(body):
    ex = int(r[iex] or 0)
    smp = int(r[ismp] or 0)
    if ex * 200 >= tot or smp * 100 >= tots:
        print(f"{n:5d} {ex:9d} {smp:6d}  {r[isrc].strip()}")
