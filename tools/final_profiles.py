"""Copy a final GPU evidence run (tools/gpu/run51.sh with P=<prefix>) into profiles/: bench lines of
cfg4 / cfg3 / cfg2 (+ the reference arm when present), the launch list, and the ncu --set full
summary of k_remedy on cfg4 (profiles/ncu_r2.md section + the traffic bench.py reads from
profiles/ncu_summary.json).  python tools/final_profiles.py <prefix>"""
import collections
import csv
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
P = sys.argv[1]
G = os.path.join(ROOT, "gpurun_out")
PR = os.path.join(ROOT, "profiles")


def last_json(path):
    line = open(path).read().strip().splitlines()[-1]
    json.loads(line)
    return line


for src, dst in (("bench", "cfg4"), ("cfg3", "cfg3"), ("cfg2", "cfg2"), ("ref", "reference")):
    f = os.path.join(G, f"{P}_{src}.log")
    if os.path.exists(f):
        open(os.path.join(PR, f"bench_r2_final_{dst}.json"), "w").write(last_json(f) + "\n")

rows = [r for r in csv.reader(open(os.path.join(G, f"{P}_launches.csv"))) if len(r) > 10]
h = rows[0]
ki, mi, vi, ui = (h.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
agg = collections.OrderedDict()
scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}
for r in rows[1:]:
    if r[mi] == "gpu__time_duration.sum":
        a = agg.setdefault(r[ki].split("(")[0][:40], [0, 0.0])
        a[0] += 1
        a[1] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1e3)
tot = sum(a[1] for a in agg.values())
table = ["| kernel | launches | total ms | share |", "|---|---|---|---|"] + [
    f"| {k} | {n} | {ms:.3f} | {ms / tot * 100:.1f}% |" for k, (n, ms) in sorted(agg.items(), key=lambda t: -t[1][1])]
shutil.copy(os.path.join(G, f"{P}_launches.csv"), os.path.join(PR, "launches_r2_final.csv"))

rep = os.path.join(G, f"{P}_prof_list_cfg4.ncu-rep")
raw = list(csv.reader(subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                                     text=True).stdout.splitlines()))
hh, units, vals = raw[0], raw[1], raw[2]
get = lambda k: vals[hh.index(k)]  # noqa: E731
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
        "smsp__thread_inst_executed_per_inst_executed.ratio", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.per_cycle_active", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"]
md = [f"- `{k}` = {get(k)} {units[hh.index(k)]}" for k in keys if k in hh]
st = {k[len("smsp__pcsamp_warps_issue_stalled_"):]: float(vals[i]) for i, k in enumerate(hh)
      if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued") and vals[i] not in ("", "n/a")}
t = sum(st.values())
md.append("- stall mix: " + ", ".join(f"{k} {x / t * 100:.1f}%" for k, x in sorted(st.items(), key=lambda a: -a[1])[:8]))
rd, wr = float(get("dram__bytes_read.sum")), float(get("dram__bytes_write.sum"))  # GB (ncu unit)
md.append(f"- DRAM per launch {rd + wr:.1f} GB = {(rd + wr) / 307.9275:.2f}x the algorithmic 307.9 GB (r2 start, 4 x 256-thread "
          f"CTAs: 945.4 GB, 3.07x)")

p = os.path.join(PR, "ncu_r2.md")
s = open(p).read()
s = s[:s.index("## Final round-2 state")] if "## Final round-2 state" in s else s
s += ("## Final round-2 state: single-device remedy at 512-thread CTAs (2 per SM), phase B member words staged "
      "CTA-wide in shared memory, warp-interleaved traversal for 2D / single-sweep 3D grids\n\n"
      "Launch list (`profiles/launches_r2_final.csv`, `python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu`; "
      "cold-cache, serialised: compare SHARES):\n\n" + "\n".join(table) +
      "\n\n### k_remedy — cfg4: 3D 512^3 checkerboard 1:100 (32^3 blocks), h=1, seed (c,c,c)\n\n"
      f"`{P}_prof_list_cfg4.ncu-rep` (`ncu --set full --clock-control none --import-source on -k regex:\"^k_remedy$\" "
      f"-s 1 -c 1`, `tools/prof_solve.py cfg4 512 2`, `P={P} bash tools/gpu/run51.sh`)\n\n" + "\n".join(md) + "\n")
open(p, "w").write(s)

js = os.path.join(PR, "ncu_summary.json")
d = json.load(open(js))
d["tag"] = f"r2 final ({P})"
d["captures"]["k_remedy"][0].update({"dram_bytes_read": rd * 1e9, "dram_bytes_write": wr * 1e9,
                                     "duration_ms": float(get("gpu__time_duration.sum")),
                                     "block_size": 512, "grid_size": int(float(get("launch__grid_size")))})
json.dump(d, open(js, "w"), indent=1)
print("\n".join(table[:4] + md))
