"""Group SASS instructions of one kernel into regions (by executed count) to see where issue slots go."""
import csv, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
seg = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "--kernel-name", f"regex:{kern}"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
hi = next(i for i, r in enumerate(rows) if len(r) > 2 and r[0] == "Address")
h = rows[hi]; I = {k: i for i, k in enumerate(h)}
data = [r for r in rows[hi + 1:] if len(r) == len(h) and r[0] != "Address"]
ex = [float(r[I["Instructions Executed"]] or 0) for r in data]
st = [float(r[I["Warp Stall Sampling (All Samples)"]] or 0) for r in data]
T, S = sum(ex), sum(st)
print(len(data), "instrs; executed", T, "samples", S)
for s in range(0, len(data), seg):
    t = sum(ex[s:s + seg]); ss = sum(st[s:s + seg])
    if t > 0.01 * T or ss > 0.02 * S:
        ops = [data[i][I["Source"]].split()[0] for i in range(s, min(s + seg, len(data))) if data[i][I["Source"]].split()]
        print(f"{s:5d} ex {t/T*100:5.1f}% stall {ss/S*100:5.1f}% maxex={max(ex[s:s+seg]):.3g} ", " ".join(ops[:16]))
