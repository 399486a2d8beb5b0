"""Copy the round's GPU outputs (gpurun_out/, written by tools/gpu/run_all.sh + run_prof.sh +
phase_times) into the tracked profiles/ summaries.  Usage: python tools/refresh_profiles.py r01"""
import csv
import json
import shutil
import subprocess
import sys

tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
G, P = "gpurun_out/", "profiles/"


def run(*cmd):
    return subprocess.run(cmd, capture_output=True, text=True).stdout


shutil.copy(G + "bench_all.jsonl", P + f"{tag}_bench_all_configs.jsonl")
shutil.copy(G + "bench_default.jsonl", P + f"{tag}_bench_default.jsonl")
shutil.copy(G + "launches_bench.csv", P + f"{tag}_ncu_launches_bench.csv")
with open(P + f"{tag}_ncu_launches_bench_summary.txt", "w") as f:
    f.write("# ncu --metrics gpu__time_duration.sum --clock-control none of: python bench.py --steps 2 --warmup 3 "
            "(default c2 workload)\n")
    f.write(run(sys.executable, "tools/launch_summary.py", G + "launches_bench.csv"))
for c in ("c2", "c4", "c4f", "c5"):
    with open(P + f"{tag}_ncu_full_{c}_summary.txt", "w") as f:
        what = "one hierarchical block launch of k_sort_fused" if c == "c4f" else "one launch of the dominant kernel"
        f.write(f"# ncu --set full --clock-control none --import-source on, {what} of "
                f"tools/prof_step.py --config {c[:2]} (same kernels and launch configuration as bench.py {c[:2]})\n")
        f.write(run(sys.executable, "tools/ncu_summary.py", G + f"full_{c}.ncu-rep"))
with open(P + f"{tag}_phase_times.txt", "w") as f:
    f.write("# tools/phase_times.py <config> (libdialsort_phase.so: -DDIALSORT_PHASE_MARKS=1), one isolated step, "
            "per-CTA %globaltimer stamps, us after the first CTA start, min/median/max over CTAs\n")
    f.write(open(G + "phase_times.txt").read())
    f.write("\n# tools/phase_radix.py (c5, n=1e8): cumulative phase ends of the slowest radix pass, us\n")
    f.write(open(G + "phase_radix.txt").read())


def metrics(rep):
    raw = run("ncu", "-i", rep, "--page", "raw", "--csv")
    rows = list(csv.reader(raw.splitlines()))
    h, u, r = rows[0], rows[1], rows[2]
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "nsecond": 1e-3, "us": 1,
            "usecond": 1, "ms": 1e3, "msecond": 1e3}

    def g(k):
        return float(r[h.index(k)].replace(",", "")) * mult[u[h.index(k)]]
    return g("dram__bytes_read.sum"), g("dram__bytes_write.sum"), g("gpu__time_duration.sum")


tr = json.load(open(P + f"{tag}_ncu_traffic.json"))
for c, k, rep in (("c2", "k_sort_fused", "c2"), ("c4", "k_part_scatter", "c4"), ("c4", "k_sort_fused", "c4f"),
                  ("c5", "k_radix_pass", "c5")):
    rd, wr, t = metrics(G + f"full_{rep}.ncu-rep")
    e = tr["configs"][c].setdefault(k, {})
    e["dram_read_bytes"], e["dram_write_bytes"], e["ncu_duration_us"] = int(rd), int(wr), round(t, 3)
json.dump(tr, open(P + f"{tag}_ncu_traffic.json", "w"), indent=1)
print("profiles refreshed")
