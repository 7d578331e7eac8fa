"""Per-instruction shared-memory wavefronts (ideal vs excessive) from an ncu source page."""
import csv, io, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO("\n".join(out.splitlines()[1:]))))
h = rows[0]
ia, isrc, iex = h.index("Address"), h.index("Source"), h.index("Instructions Executed")
iw, iwi, iwx = h.index("L1 Wavefronts Shared"), h.index("L1 Wavefronts Shared Ideal"), h.index("L1 Wavefronts Shared Excessive")
data = []
for r in rows[1:]:
    if len(r) != len(h): continue
    try:
        data.append((int(r[iw]), int(r[iwi]), int(r[iwx]), int(r[iex]), r[ia][-5:], r[isrc].strip()))
    except ValueError:
        pass
tw = sum(d[0] for d in data); tx = sum(d[2] for d in data)
print(f"total shared wavefronts {tw}, excessive {tx}")
for w, wi, wx, ex, a, s in sorted(data, reverse=True)[:40]:
    print(f"{w:10d} ideal {wi:10d} excess {wx:9d} exec {ex:9d} {a} {s[:70]}")
