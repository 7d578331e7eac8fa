"""SASS opcode mix (executed warp-instructions and stall samples) of one kernel in an ncu report.
Usage: python tools/ncu_opmix.py rep.ncu-rep [top]"""
import collections, csv, io, subprocess, sys
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
ix = hdr.index("Source"); ie = hdr.index("Instructions Executed"); iw = hdr.index("Warp Stall Sampling (All Samples)")
agg = collections.Counter(); st = collections.Counter()
for r in rows[2:]:
    if len(r) <= ie: continue
    op = r[ix].strip().split()
    if not op: continue
    o = op[1] if op[0].startswith("@") else op[0]
    try:
        agg[o] += float(r[ie] or 0); st[o] += float(r[iw] or 0)
    except ValueError:
        pass
tot = sum(agg.values()); ts = sum(st.values())
print(f"total warp-instructions {tot:.0f}, stall samples {ts:.0f}")
for o, c in agg.most_common(top):
    print(f"{o:24s} {c/tot*100:5.1f}% inst  {st[o]/ts*100:5.1f}% stall")
