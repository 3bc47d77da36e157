"""Per-rank kernel time of a C4 shard (rank 0 of `world`) on one GPU: the
kernel-side part of the strong-scaling curve (no collective)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import workloads as W  # noqa: E402
import paper_2110_03214_b200 as mp  # noqa: E402
from paper_2110_03214_b200 import dist as md  # noqa: E402

t = mp.Topology(text=W.het32_text())
p = mp.Pattern.make("full", 6)
q = md.query_tensor(0)
rec = torch.zeros(4, dtype=torch.int64, device="cuda")
base = None
for world in (1, 2, 4, 8):
    tot = 0.0
    for sel, sens in ((0, False), (1, True), (1, False)):
        for rank in range(world):
            for _ in range(3):
                mp.launch_query(t, p, sel, sens, q.data_ptr(), rec.data_ptr(), raw=True, rank=rank, world=world, busy_hint=0)
        torch.cuda.synchronize()
        worst = 0.0
        for rank in range(world):  # the step time of N ranks = the slowest rank
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(20):
                mp.launch_query(t, p, sel, sens, q.data_ptr(), rec.data_ptr(), raw=True, rank=rank, world=world, busy_hint=0)
            b.record()
            torch.cuda.synchronize()
            worst = max(worst, a.elapsed_time(b) / 20)
        tot += worst
    base = base or tot
    print(f"world {world}: slowest-rank kernels per step {tot*1e3:.1f} us  -> kernel-only speedup {base/tot:.2f}x", flush=True)

# fixed cost: the same kernel with 6 free devices (720 leaves) = launch + prologue + drain
for sel, sens in ((0, False), (1, True)):
    busy = ((1 << 32) - 1) & ~0x3F
    qq = md.query_tensor(busy)
    for _ in range(3):
        mp.launch_query(t, p, sel, sens, qq.data_ptr(), rec.data_ptr(), raw=True, busy_hint=busy)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(50):
        mp.launch_query(t, p, sel, sens, qq.data_ptr(), rec.data_ptr(), raw=True, busy_hint=busy)
    b.record()
    torch.cuda.synchronize()
    print(f"tiny query (720 leaves) sel {sel}{'s' if sens else ''}: {a.elapsed_time(b) / 50 * 1e3:.1f} us per launch (memset + kernel)")
    # full-grid launch of a tiny query: busy_hint unknown -> the grid is sized for N free
    a.record()
    for _ in range(50):
        mp.launch_query(t, p, sel, sens, qq.data_ptr(), rec.data_ptr(), raw=True)
    b.record()
    torch.cuda.synchronize()
    print(f"  same with a full grid: {a.elapsed_time(b) / 50 * 1e3:.1f} us")
