"""(Round 1; superseded by tools/summarize_r2.py, whose ncu_summary.json schema bench.py reads.) Turn ncu outputs brought back in gpurun_out/ into committed summaries under profiles/.

    python tools/summarize_profiles.py --launches gpurun_out/launches_rX.csv \
        --full gpurun_out/prof_rX.ncu-rep --tag rX --workload "<bench workload string>"
"""
import argparse, collections, csv, json, os, subprocess

ap = argparse.ArgumentParser()
ap.add_argument("--launches")
ap.add_argument("--full")
ap.add_argument("--tag", required=True)
ap.add_argument("--workload", default="")
a = ap.parse_args()
os.makedirs("profiles", exist_ok=True)
out_md = [f"# ncu summary {a.tag}\n"]
js = {"tag": a.tag, "kernels": {}}

if a.launches:
    rows = [r for r in csv.reader(open(a.launches)) if len(r) > 10]
    h = rows[0]; I = {k: i for i, k in enumerate(h)}
    tot = collections.defaultdict(float); cnt = collections.Counter()
    for r in rows[1:]:
        if r[I["Metric Name"]] != "gpu__time_duration.sum":
            continue
        name = r[I["Kernel Name"]]
        short = name.split("::")[-1].split("(")[0] if "eik" not in name else name
        for key in ("k_update", "k_remedy", "k_build", "k_prep", "k_init_active", "k_seed", "k_remedy_load", "k_local"):
            if f"::{key}<" in name or f"::{key}(" in name:
                short = key
        v = float(r[I["Metric Value"]].replace(",", ""))
        unit = r[I["Metric Unit"]]
        v = v / 1e6 if unit == "ns" else (v / 1e3 if unit == "us" else v)
        tot[short] += v; cnt[short] += 1
    T = sum(tot.values())
    out_md.append("## Launch list (`ncu --metrics gpu__time_duration.sum --clock-control none`)\n")
    out_md.append("cold-cache, serialised per-launch times; compare SHARES, not absolutes\n")
    out_md.append("| kernel | launches | total ms | share |\n|---|---|---|---|")
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        out_md.append(f"| {k} | {cnt[k]} | {v:.3f} | {v / T * 100:.1f}% |")
        js["kernels"].setdefault(k, {})["launch_list_ms_total"] = v
        js["kernels"][k]["launches"] = cnt[k]
    out_md.append("")

if a.full:
    raw = subprocess.run(["ncu", "-i", a.full, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    h = rows[0]
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
            "smsp__thread_inst_executed_per_inst_executed.ratio", "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
            "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"]
    out_md.append("## Full capture (`ncu --set full --clock-control none --import-source on`)\n")
    for r in rows[2:]:
        d = dict(zip(h, r))
        name = d["Kernel Name"]
        short = next((k for k in ("k_update", "k_remedy", "k_build") if k in name), name[:40])
        out_md.append(f"### {short}\n")
        ent = js["kernels"].setdefault(short, {})
        ent["workload"] = a.workload
        for k in keys:
            if k in d:
                out_md.append(f"- `{k}` = {d[k]}")
        st = [(k.split("stalled_")[1], float(d[k].replace(",", ""))) for k in h
              if "pcsamp_warps_issue_stalled" in k and not k.endswith("not_issued") and d[k] not in ("", "n/a")]
        t = sum(v for _, v in st)
        out_md.append("- stall mix: " + ", ".join(f"{k} {v / t * 100:.1f}%" for k, v in sorted(st, key=lambda x: -x[1])[:8]))
        mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        units = dict(zip(h, rows[1]))
        for k, nm in (("dram__bytes_read.sum", "dram_bytes_read"), ("dram__bytes_write.sum", "dram_bytes_write")):
            ent[nm] = float(d[k].replace(",", "")) * mult.get(units.get(k, "byte"), 1)
        ent["duration_ms"] = float(d["gpu__time_duration.sum"].replace(",", "")) * (1e-6 if units.get("gpu__time_duration.sum") == "ns" else 1e-3 if units.get("gpu__time_duration.sum") == "us" else 1)
        out_md.append("")
with open(f"profiles/ncu_{a.tag}.md", "w") as fh:
    fh.write("\n".join(out_md) + "\n")
with open("profiles/ncu_summary.json", "w") as fh:
    json.dump(js, fh, indent=1)
print("\n".join(out_md))
