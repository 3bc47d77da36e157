"""Deep-kernel RAW throughput probe (kernel only, CUDA events): het64 ring-7
over 40 free devices (u64 masks) and cubemesh16 ring-10 all free (u32 masks),
per selector.  python scripts/deep_rate.py"""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import workloads as W  # noqa: E402
import paper_2110_03214_b200 as mp  # noqa: E402
from paper_2110_03214_b200 import dist as md  # noqa: E402

CASES = [("het64 ring-7 (40 free, u64)", mp.Topology(text=W.het64_text()), ((1 << 64) - 1) & ~((1 << 40) - 1), 7, 40),
         ("cubemesh16 ring-10 (u32)", mp.Topology("cubemesh16"), 0, 10, 16)]
for name, t, busy, k, nf in CASES:
    p = mp.Pattern.make("ring", k)
    q = md.query64_tensor(busy)
    rec = torch.zeros(8, dtype=torch.int64, device="cuda")
    for sel, sens in ((0, False), (1, True), (1, False)):
        def f():
            mp.launch_query_wide(t, p, sel, sens, q.data_ptr(), rec.data_ptr(), busy, raw=True)
        for _ in range(2):
            f()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(3):
            f()
        b.record()
        b.synchronize()
        ms = a.elapsed_time(b) / 3
        print(f"{name} sel={sel} sens={int(sens)}: {ms:.2f} ms, {math.perm(nf, k) / ms * 1e3:.3g} emb/s", flush=True)
