"""One C5 batch launch per topology (after a warm-up) for ncu:
  ncu --set full -k regex:esa_batch -s 2 -c 2 -o gpurun_out/batch python scripts/prof_batch.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import workloads as W  # noqa: E402
import paper_2110_03214_b200 as mp  # noqa: E402
from paper_2110_03214_b200 import dist as md  # noqa: E402

SHAPE_K = [(s, k) for s in ("ring", "tree", "full") for k in range(2, 6)]
for rep in range(2):
    for name, n in (("cubemesh16", 16), ("het32", 32)):
        t = mp.Topology(name) if n == 16 else mp.Topology(text=W.het32_text())
        pats = [mp.Pattern.make(s, k) for s, k in SHAPE_K]
        pid = {sk: i for i, sk in enumerate(SHAPE_K)}
        qs = W.c5_queries(n, count=100_000)
        qt = md.queries_tensor([(q["busy"], pid[(q["shape"], q["k"])], q["selector"], q["sensitive"]) for q in qs])
        md.run_batch(t, pats, qt, raw=True)
        torch.cuda.synchronize()
