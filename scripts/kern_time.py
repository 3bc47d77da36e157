"""Per-selector C4 kernel times (RAW, het32 full-6, one stream, record
zeroed per launch): 5 repeats of 20 launches each, min / median in us.
  python scripts/kern_time.py [package_dir]"""
import math
import os
import statistics
import sys

root = sys.argv[1] if len(sys.argv) > 1 else os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, root)
import torch  # noqa: E402

import workloads as W  # noqa: E402
import paper_2110_03214_b200 as mp  # noqa: E402
from paper_2110_03214_b200 import dist as md  # noqa: E402

print("lib:", mp.LIB_PATH)
t = mp.Topology(text=W.het32_text())
p = mp.Pattern.make("full", 6)
q = md.query_tensor(0)
rec = torch.zeros(4, dtype=torch.int64, device="cuda")
for sel, sens, name in ((0, False, "greedy"), (1, True, "sens"), (1, False, "insens")):
    f = lambda: mp.launch_query(t, p, sel, sens, q.data_ptr(), rec.data_ptr(), raw=True, busy_hint=0)
    for _ in range(5):
        f()
    ts = []
    for _ in range(5):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(20):
            f()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b) / 20 * 1e3)
    print(f"{name}: min {min(ts):.1f} med {statistics.median(ts):.1f} us", flush=True)
