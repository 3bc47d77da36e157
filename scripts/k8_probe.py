"""cubemesh16, all 16 free, k = 8 RAW: narrow kernel vs the deep kernel (MAPA_F_DEEP), per shape and selector,
end to end through mapa_allocate (median of 5)."""
import math
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2110_03214_b200 as mp  # noqa: E402

t = mp.Topology("cubemesh16")
for nfree in (16, 12):
    t.set_busy(((1 << 16) - 1) & ~((1 << nfree) - 1))
    for shape in ("ring", "tree", "full"):
        p = mp.Pattern.make(shape, 8)
        for sel, sens in ((0, False), (1, True), (1, False)):
            row = []
            for deep in (False, True):
                mp.allocate(t, p, sel, sens, raw=True, deep=deep)
                ts = []
                for _ in range(5):
                    torch.cuda.synchronize()
                    t0 = time.perf_counter()
                    d = mp.allocate(t, p, sel, sens, raw=True, deep=deep)
                    ts.append(time.perf_counter() - t0)
                row.append(statistics.median(ts))
            n = math.perm(nfree, 8)
            print(f"free {nfree} {shape}-8 sel {sel}{'s' if sens else ''}: narrow {row[0]*1e3:.2f} ms "
                  f"({n/row[0]:.3g}/s)  deep {row[1]*1e3:.2f} ms ({n/row[1]:.3g}/s)", flush=True)
