"""Summarise an ncu SASS source page: top instructions by warp-stall samples."""
import csv, sys, subprocess, collections
rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "--kernel-name", f"regex:{kern}"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
hi = next(i for i, r in enumerate(rows) if len(r) > 2 and r[0] == "Address")
h = rows[hi]; data = [r for r in rows[hi + 1:] if len(r) == len(h) and r[0] != "Address"]
I = {k: i for i, k in enumerate(h)}
S = "Warp Stall Sampling (All Samples)"
tot = sum(float(r[I[S]] or 0) for r in data)
ex = "Instructions Executed"
print(kern, "samples", tot, "instr executed", sum(float(r[I[ex]] or 0) for r in data))
# opcode histogram of samples
op = collections.Counter()
for r in data:
    op[r[I["Source"]].split()[0] if r[I["Source"]].split() else "?"] += float(r[I[S]] or 0)
print("by opcode:", ", ".join(f"{k}:{v/tot*100:.1f}%" for k, v in op.most_common(12)))
order = sorted(range(len(data)), key=lambda i: -float(data[i][I[S]] or 0))[:n]
for i in sorted(order):
    r = data[i]
    print(f"{i:5d} {float(r[I[S]])/tot*100:5.1f}%  ex={r[I[ex]]:>9} {r[I['Source']].strip()[:90]}")
