"""Per-(file, line) executed instructions and stall samples of one kernel from an ncu report
(--import-source on, -lineinfo): python tools/ncu_src.py REP KERNEL_REGEX [TOP]."""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda",
                      "--kernel-name", f"regex:{kern}"], capture_output=True, text=True).stdout.splitlines()
num = lambda x: float(x) if x not in ("", "-") else 0.0
f, agg = None, {}
for r in csv.reader(out):
    if len(r) == 2 and r[0] == "File Path":
        f = r[1].split("/")[-1]
    elif len(r) > 8 and r[0].isdigit() and r[2] == "-":
        a = agg.setdefault((f, int(r[0])), [0.0, 0.0, 0.0, r[1].strip()[:80]])
        a[0] += num(r[4]); a[1] += num(r[7]); a[2] += num(r[8])
tw = sum(a[1] for a in agg.values()) or 1
ts = sum(a[0] for a in agg.values()) or 1
print(f"warp-inst {tw:.4g} thread-inst {sum(a[2] for a in agg.values()):.4g}")
byf = {}
for (fn, _), a in agg.items():
    byf[fn] = byf.get(fn, 0) + a[1]
print({k: f"{v / tw * 100:.1f}%" for k, v in byf.items()})
for (fn, l), a in sorted(agg.items(), key=lambda t: -t[1][1])[:top]:
    print(f"{fn[:14]:14s} {l:5d} ex {a[1] / tw * 100:5.1f}% thr/inst {a[2] / a[1] if a[1] else 0:5.1f} "
          f"samples {a[0] / ts * 100:5.1f}%  {a[3]}")
