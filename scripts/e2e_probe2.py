import sys, os, time, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import workloads as W
import paper_2110_03214_b200 as mp
t = mp.Topology(text=W.het32_text()); p = mp.Pattern.make("full", 6)
sels = ((0, False), (1, True), (1, False))
for _ in range(5):
    for s in sels: mp.allocate(t, p, *s, raw=True)
torch.cuda.synchronize()
per = {s: [] for s in sels}
for _ in range(30):
    for s in sels:
        t0 = time.perf_counter(); mp.allocate(t, p, *s, raw=True); per[s].append(time.perf_counter() - t0)
for s in sels: print(s, "median us", statistics.median(per[s]) * 1e6, "max", max(per[s]) * 1e6)
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
for _ in range(50): flush.zero_()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(20):
    for s in sels: mp.allocate(t, p, *s, raw=True)
print("loop avg us", (time.perf_counter() - t0) / 60 * 1e6)
