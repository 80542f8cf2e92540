"""Key raw metrics + stall breakdown of one kernel in an ncu report: python tools/ncu_raw.py REP [KERNEL_REGEX]."""
import csv
import subprocess
import sys

rep = sys.argv[1]
cmd = ["ncu", "-i", rep, "--page", "raw", "--csv"]
if len(sys.argv) > 2:
    cmd += ["--kernel-name", f"regex:{sys.argv[2]}"]
rows = list(csv.reader(subprocess.run(cmd, capture_output=True, text=True).stdout.splitlines()))
h = rows[0]
for v in rows[2:]:
    d = dict(zip(h, v))
    print(d.get("Kernel Name", "")[:60])
    for k in ("gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
              "smsp__thread_inst_executed_per_inst_executed.ratio", "smsp__issue_active.avg.pct_of_peak_sustained_active",
              "sm__warps_active.avg.per_cycle_active", "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
              "launch__registers_per_thread", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
              "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"):
        if k in d:
            print(f"  {k:55s} {d[k]}")
    st = [(k, d[k]) for k in h if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued")]
    tot = sum(float(x or 0) for _, x in st) or 1
    print("  stalls:", ", ".join(f"{k[33:]}={float(x) / tot * 100:.1f}%" for k, x in sorted(st, key=lambda t: -float(t[1] or 0))[:9]))
