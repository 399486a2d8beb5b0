"""Copy the round-2 evidence written by tools/gpu/run_round2_final.sh (gpurun_out/r02_*) into the
tracked profiles/ and refresh profiles/r02_ncu_traffic.json (DRAM bytes per launch of each
captured kernel, read by bench.py's roofline `traffic`)."""
import glob
import json
import os
import re
import shutil
import subprocess
import sys

G, P = "gpurun_out/", "profiles/"
copied = []
for pat in ("r02_bench_default.jsonl", "r02_bench_all.jsonl", "r02_bench_c2_single.jsonl", "r02_bench_c4_exact.jsonl",
            "r02_paper_grid.jsonl", "r02_rank_step.jsonl", "r02_phase_c2.txt", "r02_launches_bench.csv",
            "r02_ncu_*_summary.txt", "r02_ncu_*_hot.txt"):
    for f in glob.glob(G + pat):
        dst = P + {"r02_bench_all.jsonl": "r02_bench_all_configs.jsonl", "r02_launches_bench.csv": "r02_ncu_launches_bench.csv",
                   "r02_bench_c2_single.jsonl": "r02_bench_c2_single_call.jsonl"}.get(os.path.basename(f), os.path.basename(f))
        shutil.copy(f, dst)
        copied.append(dst)
if os.path.exists(G + "r02_launches_bench.csv"):
    out = subprocess.run([sys.executable, "tools/launch_summary.py", G + "r02_launches_bench.csv"], capture_output=True,
                         text=True).stdout
    with open(P + "r02_ncu_launches_bench_summary.txt", "w") as f:
        f.write("# ncu --metrics gpu__time_duration.sum --clock-control none of: python bench.py --steps 64 --warmup 32 "
                "--no-cpu-baseline --no-e2e (default c2 workload, 32 steps per k_sort_batch launch)\n")
        f.write(out)

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "us": 1, "usecond": 1, "ms": 1e3, "msecond": 1e3,
        "ns": 1e-3, "nsecond": 1e-3}


def parse(path):
    vals, kern = {}, None
    for line in open(path):
        if line.startswith("=="):
            kern = line[3:].strip()
        m = re.match(r"\s+(\S+)\s+([\d.]+) (\S+)", line)
        if m and m.group(3) in UNIT:
            vals[m.group(1)] = float(m.group(2)) * UNIT[m.group(3)]
    return kern, vals


KID = {"k_part_place": "k_part_place_est"}  # profiler name of the captured launch (sampled schedule)
tr = json.load(open(P + "r02_ncu_traffic.json"))
for f in glob.glob(P + "r02_ncu_*_summary.txt"):
    m = re.match(r"r02_ncu_(.+?)_(k_[a-z_0-9]+)_summary.txt", os.path.basename(f))
    if not m or m.group(2) == "k_part_scatter":
        continue
    cfg, k = m.group(1), KID.get(m.group(2), m.group(2))
    kern, v = parse(f)
    if "dram__bytes_read.sum" not in v:
        continue
    e = tr["configs"].setdefault(cfg, {}).setdefault(k, {})
    e["dram_read_bytes"] = int(v["dram__bytes_read.sum"])
    e["dram_write_bytes"] = int(v["dram__bytes_write.sum"])
    e["ncu_duration_us"] = round(v["gpu__time_duration.sum"], 3)
    e["ncu_kernel"] = kern
json.dump(tr, open(P + "r02_ncu_traffic.json", "w"), indent=1)
print("copied", len(copied), "files; traffic entries:", {c: list(d) for c, d in tr["configs"].items()})
