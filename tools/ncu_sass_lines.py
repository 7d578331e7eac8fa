import csv, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
cur = None; hdr = None; data = []
for r in rows:
    if not r: continue
    if r[0] == "Line No": hdr = r; continue
    if hdr is None: continue
    if r[0] != "": cur = (r[0], r[1].strip()[:70]); continue
    try: s = int(r[4] or 0); e = int(r[7] or 0)
    except: continue
    data.append((s, e, r[3].strip()[:50], cur))
ts = sum(d[0] for d in data); te = sum(d[1] for d in data)
print("samples", ts, "warp-inst", te)
import collections
byline = collections.defaultdict(lambda: [0, 0])
for s, e, src, cur in data:
    byline[cur][0] += s; byline[cur][1] += e
print("-- by source line (inst share, sample share)")
for cur, (s, e) in sorted(byline.items(), key=lambda kv: -kv[1][1])[:30]:
    print(f"{100*e/te:5.1f}% inst {100*s/ts:5.1f}% smp  {cur}")
