"""One C4 launch per selector (RAW, het32 x full-6) for ncu captures:
  ncu --set full --import-source on -k regex:esa_single -c 3 -o gpurun_out/x python scripts/prof_one.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import workloads as W  # noqa: E402
import paper_2110_03214_b200 as mp  # noqa: E402
from paper_2110_03214_b200 import dist as md  # noqa: E402

t = mp.Topology(text=W.het32_text())
pat = mp.Pattern.make("full", int(os.environ.get("PROF_K", "6")))
for sel, sens in ((0, False), (1, True), (1, False)):
    rec, q = md.run_query(t, pat, sel, sens, 0, raw=True)
    torch.cuda.synchronize()
    print(sel, sens, md.records_from_tensor(rec)[0].leaves)
