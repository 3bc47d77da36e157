"""Deep-kernel launches for ncu: cubemesh16 ring-PROF_K (default 10), Greedy,
RAW then canonical, each twice (skip the first pair with ncu -s 2):
  ncu --set full --import-source on -k regex:esa_deep -s 2 -c 2 -o gpurun_out/deep python scripts/prof_deep.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2110_03214_b200 as mp  # noqa: E402
from paper_2110_03214_b200 import dist as md  # noqa: E402

t = mp.Topology(os.environ.get("PROF_TOPO", "cubemesh16"))
pat = mp.Pattern.make(os.environ.get("PROF_SHAPE", "ring"), int(os.environ.get("PROF_K", "10")))
sel, sens = int(os.environ.get("PROF_SEL", "0")), bool(int(os.environ.get("PROF_SENS", "0")))
for _ in range(2):
    for raw in (True, False):
        rec, q = md.run_query_wide(t, pat, sel, sens, 0, raw=raw)
        torch.cuda.synchronize()
        print(raw, md.wide_records_from_tensor(rec)[0].leaves)
