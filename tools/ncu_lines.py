"""Aggregate ncu SASS metrics by CUDA source line (needs -lineinfo + --import-source).
Usage: python tools/ncu_lines.py rep.ncu-rep [top]"""
import collections, csv, io, subprocess, sys
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
agg = collections.defaultdict(lambda: [0.0, 0.0, 0.0, ""])
cur_file = "?"; hdr = None
for r in csv.reader(io.StringIO(out)):
    if not r: continue
    if r[0] == "File Path": cur_file = r[1].split("/")[-1]; continue
    if r[0] == "Function Name": continue
    if r[0] == "Line No": hdr = r; continue
    if hdr is None or len(r) < 8: continue
    try:
        s = float(r[4] or 0); i = float(r[7] or 0)
    except ValueError:
        continue
    key = (cur_file, r[0])
    a = agg[key]; a[0] += s; a[1] += i
    if r[1].strip(): a[3] = r[1].strip()
tot = sum(a[0] for a in agg.values()) or 1
toti = sum(a[1] for a in agg.values()) or 1
print(f"total stall samples {tot:.0f}, warp-instructions {toti:.0f}")
for (f, ln), a in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{100*a[0]/tot:5.1f}% smp {100*a[1]/toti:5.1f}% inst  {f}:{ln:5s} {a[3][:80]}")
