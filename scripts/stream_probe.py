"""C4 step (one RAW query per selector) with the three launches on ONE stream
vs on three streams (prologues / tails overlap), for rank 0 of world 1 / 2 /
4 / 8: kernel-side strong-scaling probe (no collective)."""
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
main = torch.cuda.current_stream()
side = [torch.cuda.Stream() for _ in range(3)]


def step(world, rank, multi):
    recs.zero_()  # one memset per step; the launches carry MAPA_F_ZEROED
    if not multi:
        for i, (sel, sens) in enumerate(SELS):
            mp.launch_query(t, p, sel, sens, q.data_ptr(), recs[i].data_ptr(), raw=True, rank=rank, world=world,
                            busy_hint=0, stream=main, zeroed=True)
        return
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


base = {}
for multi in (False, True):
    for world in (1, 2, 4, 8):
        worst = 0.0
        for rank in range(world):
            for _ in range(3):
                step(world, rank, multi)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(main)
            for _ in range(20):
                step(world, rank, multi)
            b.record(main)
            torch.cuda.synchronize()
            worst = max(worst, a.elapsed_time(b) / 20)
        base.setdefault(multi, worst)
        print(f"{'3 streams' if multi else '1 stream '} world {world}: slowest rank {worst*1e3:.1f} us/step -> "
              f"{base[False] / worst:.2f}x of 1 stream world 1", flush=True)
