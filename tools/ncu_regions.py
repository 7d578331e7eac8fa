"""Split an ncu SASS source page into regions at BAR.SYNC / loop labels and sum
stall samples and executed instructions per region.  Usage: ncu_regions.py rep"""
import csv, io, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO("\n".join(out.splitlines()[1:]))))
h = rows[0]
ia, isrc, ismp, iex = (h.index(k) for k in ["Address", "Source", "Warp Stall Sampling (All Samples)", "Instructions Executed"])
data = [(int(r[ia], 16), r[isrc].strip(), int(r[ismp]), int(r[iex])) for r in rows[1:] if len(r) == len(h)]
cuts = [a for a, s, _, _ in data if "BAR.SYNC" in s or "EXIT" in s]
print("barriers/exits at", [hex(c & 0xffff) for c in cuts])
reg = 0
acc = {}
for a, s, smp, ex in data:
    acc.setdefault(reg, [0, 0, a, a])
    acc[reg][0] += smp; acc[reg][1] += ex; acc[reg][3] = a
    if a in cuts:
        reg += 1
tot = sum(v[0] for v in acc.values())
for r, (smp, ex, a0, a1) in acc.items():
    print(f"region {r}: {hex(a0 & 0xffff)}-{hex(a1 & 0xffff)} samples {100*smp/tot:5.1f}% instr {ex}")
