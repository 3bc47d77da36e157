"""C3-style kernel times: cubemesh16 (W = 16), k = 8 RAW queries with 16 / 14 / 12
free devices, per shape and selector (5 repeats of 20 launches, median, us).
  python scripts/kern_time16.py [package_root]"""
import math
import os
import statistics
import sys

sys.path.insert(0, sys.argv[1] if len(sys.argv) > 1 else os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2110_03214_b200 as mp  # noqa: E402
from paper_2110_03214_b200 import dist as md  # noqa: E402

t = mp.Topology("cubemesh16")
rec = torch.zeros(4, dtype=torch.int64, device="cuda")
for nfree in (16, 14, 12):
    busy = ((1 << 16) - 1) & ~((1 << nfree) - 1)
    q = md.query_tensor(busy)
    for shape in ("ring", "full"):
        p = mp.Pattern.make(shape, 8)
        row = []
        for sel, sens in ((0, False), (1, True), (1, False)):
            f = lambda: mp.launch_query(t, p, sel, sens, q.data_ptr(), rec.data_ptr(), raw=True, busy_hint=busy)
            for _ in range(3):
                f()
            ts = []
            for _ in range(5):
                torch.cuda.synchronize()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                for _ in range(20):
                    f()
                b.record()
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b) / 20 * 1e3)
            row.append(statistics.median(ts))
        n = math.perm(nfree, 8)
        print(f"free {nfree} {shape}-8: greedy {row[0]:.1f} sens {row[1]:.1f} insens {row[2]:.1f} us "
              f"({n / row[0] / 1e6:.3g} / {n / row[1] / 1e6:.3g} / {n / row[2] / 1e6:.3g} e12 embeddings/s)", flush=True)
