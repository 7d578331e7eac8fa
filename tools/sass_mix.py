"""Static SASS opcode mix of the fast kernels in libtgk.so (cuobjdump -sass):
per kernel instance the instruction count by opcode, with the mnemonics that
show the Blackwell data movement (UBLKCP = cp.async.bulk TMA copies, SYNCS =
mbarrier, LDGSTS = cp.async, LDS/STS shared memory, DFMA/DADD/DMUL FP64).
Usage: python tools/sass_mix.py [kernel-substring ...]"""
import collections
import os
import re
import subprocess
import sys

LIB = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2602_05052_b200", "lib",
                   "libtgk.so")
WANT = sys.argv[1:] or ["k_fast_scalarILi2ELi0ELb1ELi1E", "k_fast_scalarILi2ELi0ELb0ELi1E", "k_fast_elastILi2ELi0ELi1E"]
out = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
funcs, cur = collections.OrderedDict(), None
for line in out.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        cur = m.group(1)
        funcs[cur] = collections.Counter()
        continue
    m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", line)
    if cur and m:
        funcs[cur][m.group(1)] += 1
for name, mix in funcs.items():
    if not any(w in name for w in WANT):
        continue
    total = sum(mix.values())
    print(f"== {name}\n   {total} instructions")
    for op, n in mix.most_common(40):
        print(f"   {op:10s} {n:6d}")
    for op in ["UBLKCP", "SYNCS", "LDGSTS", "UTMALDG"]:
        print(f"   [{op}: {mix.get(op, 0)}]")
