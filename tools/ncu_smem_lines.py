"""Shared-memory wavefronts (actual vs ideal) per CUDA source line from an ncu report."""
import collections, csv, io, subprocess, sys
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
agg = collections.defaultdict(lambda: [0.0, 0.0, ""]); cur = "?"; hdr = None
for r in csv.reader(io.StringIO(out)):
    if not r: continue
    if r[0] == "File Path": cur = r[1].split("/")[-1]; continue
    if r[0] == "Function Name": continue
    if r[0] == "Line No": hdr = r; iw = hdr.index("L1 Wavefronts Shared"); ii = hdr.index("L1 Wavefronts Shared Ideal"); continue
    if hdr is None or r[0] == "": continue   # CUDA-line rows only (SASS rows have no line number)
    try: w = float(r[iw] or 0); wi = float(r[ii] or 0)
    except (ValueError, IndexError): continue
    a = agg[(cur, r[0])]; a[0] += w; a[1] += wi; a[2] = r[1].strip()
tot = sum(a[0] for a in agg.values()) or 1
print(f"total shared wavefronts {tot:.3e} (ideal {sum(a[1] for a in agg.values()):.3e})")
for (f, ln), a in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{100*a[0]/tot:5.1f}%  {a[0]:.2e} (ideal {a[1]:.2e})  {f}:{ln:5s} {a[2][:70]}")
