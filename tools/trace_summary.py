import glob, sys
import numpy as np
for f in sorted(glob.glob(sys.argv[1] if len(sys.argv) > 1 else 'gpurun_out/trace_*.bin')):
    t = np.fromfile(f, dtype=np.int64).reshape(-1, 8)
    start, pro, a, b, epi, sm, nch, end = t.T
    dur = end - start
    print(f"{f.split('trace_')[1][:-4]:10s} blocks {len(t)} blk {dur.mean():6.0f}cyc pro {pro.mean():6.0f} A {a.mean():6.0f} ({a.mean()/nch.mean():5.0f}/ch) B {b.mean():6.0f} ({b.mean()/nch.mean():5.0f}/ch) epi {epi.mean():5.0f} nch {nch.mean():5.2f}")
