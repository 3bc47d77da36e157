"""ncu target: the C4 kernels on a tiny query (6 free devices, 720 leaves):
the fixed per-launch cost (prologue, context, drain)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import workloads as W  # noqa: E402
import paper_2110_03214_b200 as mp  # noqa: E402
from paper_2110_03214_b200 import dist as md  # noqa: E402

t = mp.Topology(text=W.het32_text())
p = mp.Pattern.make("full", 6)
busy = ((1 << 32) - 1) & ~0x3F
q = md.query_tensor(busy)
rec = torch.zeros(4, dtype=torch.int64, device="cuda")
for sel, sens in ((0, False), (1, True), (1, False)):
    for _ in range(2):
        mp.launch_query(t, p, sel, sens, q.data_ptr(), rec.data_ptr(), raw=True, busy_hint=0)
    torch.cuda.synchronize()
