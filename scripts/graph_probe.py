"""C4 step strong-scaling probe (kernel side, virtual ranks on one GPU): the
three selector launches of rank 0..world-1 on three streams, enqueued by the
host every step vs replayed from a CUDA graph captured once per (world, rank).
The slowest rank's step time vs world 1 (no collective)."""
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
recs = torch.zeros((3, 4), dtype=torch.int64, device="cuda")
SELS = ((0, False), (1, True), (1, False))
side = [torch.cuda.Stream() for _ in range(3)]


def step(world, rank, main):
    recs.zero_()  # one memset per step; the launches carry MAPA_F_ZEROED
    ev = torch.cuda.Event()
    ev.record(main)
    for i, (sel, sens) in enumerate(SELS):
        side[i].wait_event(ev)
        mp.launch_query(t, p, sel, sens, q.data_ptr(), recs[i].data_ptr(), raw=True, rank=rank, world=world,
                        busy_hint=0, stream=side[i], zeroed=True)
    for s in side:
        e2 = torch.cuda.Event()
        e2.record(s)
        main.wait_event(e2)


def timed(fn, main, n=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(main)
    for _ in range(n):
        fn()
    b.record(main)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


base = None
for mode in ("host", "graph"):
    for world in (1, 2, 4, 8):
        worst = 0.0
        for rank in range(world):
            main = torch.cuda.current_stream()
            if mode == "host":
                ms = timed(lambda: step(world, rank, main), main)
            else:
                cap = torch.cuda.Stream()
                for _ in range(3):
                    step(world, rank, cap)  # warm the caches outside the capture
                torch.cuda.synchronize()
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=cap):
                    step(world, rank, cap)
                ms = timed(g.replay, main)
            worst = max(worst, ms)
        base = base or worst
        print(f"{mode:5s} world {world}: slowest rank {worst*1e3:.1f} us/step -> {base / worst:.2f}x", flush=True)
