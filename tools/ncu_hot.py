"""Summarise an ncu source page (SASS): hottest instructions by stall samples,
and executed-instruction mix by opcode.  Usage: python tools/ncu_hot.py rep.ncu-rep [N]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
lines = out.splitlines()
rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
h = rows[0]
ix = {k: h.index(k) for k in ["Address", "Source", "Warp Stall Sampling (All Samples)", "Instructions Executed"]}
data = []
for r in rows[1:]:
    if len(r) < len(h):
        continue
    try:
        data.append((int(r[ix["Warp Stall Sampling (All Samples)"]]), int(r[ix["Instructions Executed"]]),
                     r[ix["Address"]], r[ix["Source"]].strip()))
    except ValueError:
        pass
tot_s = sum(d[0] for d in data)
tot_i = sum(d[1] for d in data)
print(f"total samples {tot_s}, warp-instructions executed {tot_i}")
mix = collections.Counter()
smp = collections.Counter()
for s, i, a, src in data:
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    op = op.split(".")[0]
    mix[op] += i
    smp[op] += s
print("opcode mix (warp-instr executed, stall samples):")
for op, n in mix.most_common(25):
    print(f"  {op:10s} {n:12d} {100*n/tot_i:5.1f}%  samples {100*smp[op]/max(1,tot_s):5.1f}%")
print("hottest instructions:")
for s, i, a, src in sorted(data, reverse=True)[:top]:
    print(f"  {100*s/max(1,tot_s):5.2f}% {i:10d} {a[-5:]} {src[:90]}")
