"""Per-CUDA-source-line warp-stall samples of one kernel from an ncu report
(--import-source on, -lineinfo): python tools/ncu_lines.py REP KERNEL_REGEX [TOP]."""
import csv
import subprocess
import sys
from collections import defaultdict

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda",
                      "--kernel-name", f"regex:{kern}"], capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
samples, execd, text, stalls = defaultdict(float), defaultdict(float), {}, defaultdict(lambda: defaultdict(float))
hdr = None
for r in rows:
    if len(r) > 4 and r[0] == "Line No":
        hdr = {k: i for i, k in enumerate(r)}
        snames = [k for k in r if k.startswith("stall_") and "Not Issued" not in k]
        continue
    if hdr is None or len(r) < len(hdr) or not r[0].isdigit():
        continue
    ln = int(r[0])
    text[ln] = r[1].strip()
    try:
        samples[ln] += float(r[4] or 0)
        execd[ln] += float(r[7] or 0)
        for k in snames:
            stalls[ln][k] += float(r[hdr[k]] or 0)
    except ValueError:
        pass
S = sum(samples.values())
E = sum(execd.values())
print(f"samples {S:.0f} executed {E:.3g}")
for ln, v in sorted(samples.items(), key=lambda kv: -kv[1])[:top]:
    st = sorted(stalls[ln].items(), key=lambda kv: -kv[1])[:3]
    sts = " ".join(f"{k[6:]}={x / max(v, 1) * 100:.0f}%" for k, x in st if x > 0)
    print(f"{ln:5d} {v / S * 100:5.1f}% ex {execd[ln] / max(E, 1) * 100:5.1f}%  {sts:40s} {text[ln][:90]}")

if len(sys.argv) > 4:  # region sums: name=lo-hi,...
    for spec in sys.argv[4].split(","):
        nm, rg = spec.split("=")
        lo, hi = map(int, rg.split("-"))
        s = sum(v for l, v in samples.items() if lo <= l <= hi)
        e = sum(v for l, v in execd.items() if lo <= l <= hi)
        print(f"region {nm:10s} samples {s / S * 100:5.1f}%  executed {e / E * 100:5.1f}%  ({e:.3g} warp instr)")
