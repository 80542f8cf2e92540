"""Round-2 ncu summaries: launch list + full captures (one kernel each) -> profiles/ncu_r2.md and the
machine-readable profiles/ncu_summary.json (bench.py reads `traffic` from its captures).

    python tools/summarize_r2.py --launches gpurun_out/launches_r2.csv \
        --full gpurun_out/prof_list_cfg4.ncu-rep k_remedy "<workload>" ... --tag r2

Besides the usual counters it reports the lane efficiency (thread instructions per warp
instruction, out of 32) of the compaction code, from the per-line source page of a capture made
with -lineinfo / --import-source on: phase B of the member-list remedy (rem_members) and the update
step's next-list reservation and appends (block_reserve + the append loop).
"""
import argparse
import collections
import csv
import json
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "paper_2106_15869_b200", "csrc", "eik_ifim.cu")


def line_range(pattern_start, pattern_end, src=SRC):
    """First line matching pattern_start .. the next line matching pattern_end (1-based, inclusive)."""
    lines = open(src).read().splitlines()
    a = next(i for i, l in enumerate(lines) if re.search(pattern_start, l))
    b = next(i for i in range(a + 1, len(lines)) if re.search(pattern_end, lines[i]))
    return a + 1, b + 1


def source_lines(rep, kernel):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda",
                          "--kernel-name", f"regex:{kernel}"], capture_output=True, text=True).stdout.splitlines()
    num = lambda x: float(x) if x not in ("", "-") else 0.0  # noqa: E731
    f, agg = None, {}
    for r in csv.reader(out):
        if len(r) == 2 and r[0] == "File Path":
            f = os.path.basename(r[1])
        elif len(r) > 8 and r[0].isdigit() and r[2] == "-":
            a = agg.setdefault((f, int(r[0])), [0.0, 0.0, 0.0])
            a[0] += num(r[4])  # stall samples
            a[1] += num(r[7])  # warp instructions executed
            a[2] += num(r[8])  # thread instructions executed
    return agg


def lane_eff(agg, fname, lo, hi):
    w = sum(v[1] for (f, l), v in agg.items() if f == fname and lo <= l <= hi)
    t = sum(v[2] for (f, l), v in agg.items() if f == fname and lo <= l <= hi)
    tot = sum(v[1] for v in agg.values()) or 1.0
    return (t / w if w else 0.0), w / tot


KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
        "smsp__thread_inst_executed_per_inst_executed.ratio", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.per_cycle_active", "launch__registers_per_thread", "launch__grid_size",
        "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"]
MULT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--full", nargs=3, action="append", default=[], metavar=("REP", "KERNEL", "WORKLOAD"))
    ap.add_argument("--tag", required=True)
    a = ap.parse_args()
    md = [f"# ncu summary {a.tag}\n"]
    js_path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    js = {"tag": a.tag, "kernels": {}, "captures": {}}
    if a.launches:
        rows = [r for r in csv.reader(open(a.launches)) if len(r) > 10]
        h = rows[0]
        I = {k: i for i, k in enumerate(h)}
        tot, cnt = collections.defaultdict(float), collections.Counter()
        for r in rows[1:]:
            if r[I["Metric Name"]] != "gpu__time_duration.sum":
                continue
            name = r[I["Kernel Name"]]
            m = re.search(r"::(k_[a-z0-9_]+)[<(]", name)
            short = m.group(1) if m else name.split("(")[0][-40:]
            v = float(r[I["Metric Value"]].replace(",", ""))
            unit = r[I["Metric Unit"]]
            v = v / 1e6 if unit == "ns" else (v / 1e3 if unit == "us" else v)
            tot[short] += v
            cnt[short] += 1
        T = sum(tot.values())
        md.append("## Launch list (`ncu --metrics gpu__time_duration.sum --clock-control none`, "
                  "`python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu`)\n")
        md.append("cold-cache, serialised per-launch times; compare SHARES, not absolutes\n")
        md.append("| kernel | launches | total ms | share |\n|---|---|---|---|")
        for k, v in sorted(tot.items(), key=lambda x: -x[1]):
            md.append(f"| {k} | {cnt[k]} | {v:.3f} | {v / T * 100:.1f}% |")
            js["kernels"][k] = {"launch_list_ms_total": v, "launches": cnt[k]}
        md.append("")
    md.append("## Full captures (`ncu --set full --clock-control none --import-source on`, one launch each)\n")
    brs_lo, brs_hi = line_range(r"^__device__ __forceinline__ unsigned block_reserve", r"^}")
    pb_lo, pb_hi = line_range(r"^__device__ __forceinline__ void rem_members", r"^}")
    app_lo, app_hi = line_range(r"unsigned pos = block_reserve<MR>\(tot, lenN", r"^        }$")
    for rep, kernel, workload in a.full:
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(raw.splitlines()))
        h, units = rows[0], dict(zip(rows[0], rows[1]))
        d = dict(zip(h, rows[2]))
        md.append(f"### {kernel} — {workload}\n")
        md.append(f"`{os.path.basename(rep)}`\n")
        for k in KEYS:
            if k in d:
                md.append(f"- `{k}` = {d[k]} {units.get(k, '')}".rstrip())
        st = [(k.split("stalled_")[1], float(d[k].replace(",", ""))) for k in h
              if "pcsamp_warps_issue_stalled" in k and not k.endswith("not_issued") and d[k] not in ("", "n/a")]
        t = sum(v for _, v in st) or 1.0
        md.append("- stall mix: " + ", ".join(f"{k} {v / t * 100:.1f}%" for k, v in sorted(st, key=lambda x: -x[1])[:8]))
        ent = {"workload": workload}
        for k, nm in (("dram__bytes_read.sum", "dram_bytes_read"), ("dram__bytes_write.sum", "dram_bytes_write")):
            ent[nm] = float(d[k].replace(",", "")) * MULT.get(units.get(k, "byte"), 1)
        tu = units.get("gpu__time_duration.sum")
        ent["duration_ms"] = float(d["gpu__time_duration.sum"].replace(",", "")) * (
            1e-6 if tu == "ns" else 1e-3 if tu == "us" else 1.0)
        agg = source_lines(rep, kernel)
        if agg:
            if kernel == "k_remedy":
                e, share = lane_eff(agg, "eik_ifim.cu", pb_lo, pb_hi)
                md.append(f"- compaction (phase B, `rem_members`, eik_ifim.cu:{pb_lo}-{pb_hi}): "
                          f"{e:.2f} active lanes per warp instruction ({e / 32 * 100:.1f} %), "
                          f"{share * 100:.1f} % of the kernel's warp instructions")
                ent["compaction_lanes_per_inst"] = round(e, 2)
            if kernel == "k_update":
                e1, s1 = lane_eff(agg, "eik_ifim.cu", brs_lo, brs_hi)
                e2, s2 = lane_eff(agg, "eik_ifim.cu", app_lo, app_hi)
                md.append(f"- compaction (next-list reservation `block_reserve`, eik_ifim.cu:{brs_lo}-{brs_hi}): "
                          f"{e1:.2f} lanes per warp instruction ({e1 / 32 * 100:.1f} %), {s1 * 100:.1f} % of instructions")
                md.append(f"- compaction (next-list appends, eik_ifim.cu:{app_lo}-{app_hi}): "
                          f"{e2:.2f} lanes per warp instruction ({e2 / 32 * 100:.1f} %), {s2 * 100:.1f} % of instructions")
                ent["compaction_lanes_per_inst"] = round(e1, 2)
                ent["append_lanes_per_inst"] = round(e2, 2)
        js["captures"].setdefault(kernel, []).append(ent)
        md.append("")
    with open(os.path.join(ROOT, "profiles", f"ncu_{a.tag}.md"), "w") as fh:
        fh.write("\n".join(md) + "\n")
    with open(js_path, "w") as fh:
        json.dump(js, fh, indent=1)
    print("\n".join(md))


if __name__ == "__main__":
    main()
