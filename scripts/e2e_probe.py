import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes, torch
import workloads as W
import paper_2110_03214_b200 as mp
from paper_2110_03214_b200 import dist as md
t = mp.Topology(text=W.het32_text()); p = mp.Pattern.make("full", 6)
for _ in range(5): mp.allocate(t, p, 0, False, raw=True)
torch.cuda.synchronize()
N=50
t0=time.perf_counter()
for _ in range(N): mp.allocate(t, p, 0, False, raw=True)
t1=time.perf_counter(); print("python mp.allocate us", (t1-t0)/N*1e6)
d = mp.Decision(); s = torch.cuda.current_stream().cuda_stream
t0=time.perf_counter()
for _ in range(N): mp._lib.mapa_allocate(t.handle, p.handle, 0, 0, 2, s, ctypes.byref(d))
t1=time.perf_counter(); print("raw ctypes mapa_allocate us", (t1-t0)/N*1e6)
t0=time.perf_counter()
for _ in range(N): mp._lib.mapa_allocate(t.handle, p.handle, 0, 0, 2, None, ctypes.byref(d))
t1=time.perf_counter(); print("raw ctypes default stream us", (t1-t0)/N*1e6)
q = md.query_tensor(0); rec = torch.empty(4, dtype=torch.int64, device="cuda")
torch.cuda.synchronize()
t0=time.perf_counter()
for _ in range(N):
    mp._lib.mapa_launch_query(t.handle, p.handle, 0, 0, q.data_ptr(), rec.data_ptr(), 2, 0, 1, 0, s)
torch.cuda.synchronize()
t1=time.perf_counter(); print("launch_query back-to-back us", (t1-t0)/N*1e6)
a,b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(N):
    mp._lib.mapa_launch_query(t.handle, p.handle, 0, 0, q.data_ptr(), rec.data_ptr(), 2, 0, 1, 0, s)
b.record(); torch.cuda.synchronize(); print("device per launch us", a.elapsed_time(b)/N*1e3)
