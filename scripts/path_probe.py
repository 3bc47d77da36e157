"""Narrow vs deep kernel throughput (device events) on cubemesh16, all free and
half busy, k = 5..8, RAW, the three selectors: where should mapa_allocate route?"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2110_03214_b200 as mp  # noqa: E402
from paper_2110_03214_b200 import dist as md  # noqa: E402


def timed(fn, n=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


t = mp.Topology("cubemesh16")
for busy in (0, 0b0000001100000011):
    for shape in ("ring", "full"):
        for k in (5, 6, 7, 8):
            p = mp.Pattern.make(shape, k)
            out = []
            for sel, sens in ((0, False), (1, True)):
                q = md.query_tensor(busy, 0, sel, sens)
                rec = torch.zeros(4, dtype=torch.int64, device="cuda")
                q64 = md.query64_tensor(busy, sel, sens)
                rec8 = torch.zeros(8, dtype=torch.int64, device="cuda")
                tn = timed(lambda: mp.launch_query(t, p, sel, sens, q.data_ptr(), rec.data_ptr(), raw=True, busy_hint=busy))
                td = timed(lambda: mp.launch_query_wide(t, p, sel, sens, q64.data_ptr(), rec8.data_ptr(), busy, raw=True))
                out.append(f"sel{sel}{'s' if sens else ''} narrow {tn*1e3:8.1f} us deep {td*1e3:8.1f} us")
            print(f"busy {busy:#06x} {shape}-{k}: " + " | ".join(out), flush=True)
