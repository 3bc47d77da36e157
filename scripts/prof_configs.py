"""ncu target: one launch of the dominant kernel of every bench config, in a
fixed order (index -> config in KERNELS below):
  0-2  C4   esa_single<32,6,*>   het32 full-6 RAW: Greedy, Preserve-sensitive, Preserve-insensitive
  3    C1   esa_batch<8>         1e5 dgx1v ring-3 queries
  4    C2   esa_trace<8>         dgx1p 1000-job Preserve trace
  5    C3   esa_single<16,8,*>   one cubemesh16 k=8 C3 query (the heaviest of the first 50)
  6    C5   esa_batch<32>        1e5 het32 C5 queries
  7    deep esa_deep             cubemesh16 ring-10 RAW Greedy
  ncu --set full -k regex:esa_ -o gpurun_out/x python scripts/prof_configs.py
then: python scripts/ncu_summary.py --rep gpurun_out/x.ncu-rep --tag r02 --configs"""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import workloads as W  # noqa: E402
import paper_2110_03214_b200 as mp  # noqa: E402
from paper_2110_03214_b200 import dist as md  # noqa: E402

KERNELS = ["c4_greedy", "c4_preserve_sensitive", "c4_preserve_insensitive", "c1", "c2", "c3", "c5", "deep"]
SHAPE_K = [(s, k) for s in ("ring", "tree", "full") for k in range(2, 6)]

def main():
    t = mp.Topology(text=W.het32_text())
    p = mp.Pattern.make("full", 6)
    q = md.query_tensor(0)
    rec = torch.zeros(4, dtype=torch.int64, device="cuda")
    for sel, sens in ((0, False), (1, True), (1, False)):
        mp.launch_query(t, p, sel, sens, q.data_ptr(), rec.data_ptr(), raw=True, busy_hint=0)
        torch.cuda.synchronize()
    # C1
    t8 = mp.Topology("dgx1v")
    rows = [(0, 0, [0, 1, 1][i % 3], [0, 1, 0][i % 3]) for i in range(100_000)]
    md.run_batch(t8, [mp.Pattern.make("ring", 3)], md.queries_tensor(rows), raw=True)
    torch.cuda.synchronize()
    # C2
    jobs = W.c2_jobs(2110 + 5, 1000)
    ops = W.fifo_ops(jobs, 8)
    pid = {sk: i for i, sk in enumerate(SHAPE_K)}
    pats = [mp.Pattern.make(s, k) for s, k in SHAPE_K]
    dops = torch.tensor([[o, j] for o, j in ops], dtype=torch.int32, device="cuda").reshape(1, -1, 2)
    djobs = torch.tensor([[0, pid[(j["shape"], j["k"])], 1, j["sensitive"]] for j in jobs], dtype=torch.int32,
                         device="cuda").reshape(1, -1, 4)
    md.run_trace(mp.Topology("dgx1p"), pats, dops, djobs)
    torch.cuda.synchronize()
    # C3: the heaviest of the bench's first 50 k=8 queries
    qs = [x for x in W.c3_queries(per_case=1000) if x["k"] == 8][:50]
    x = max(qs, key=lambda x: math.perm(16 - bin(x["busy"]).count("1"), 8) if 16 - bin(x["busy"]).count("1") >= 8 else 0)
    t16 = mp.Topology("cubemesh16")
    md.run_queries(t16, [mp.Pattern.make(x["shape"], 8)], [(x["busy"], 0, x["selector"], x["sensitive"])], raw=True)
    torch.cuda.synchronize()
    # C5 het32
    c5 = W.c5_queries(32, count=100_000)
    qt = md.queries_tensor([(c["busy"], pid[(c["shape"], c["k"])], c["selector"], c["sensitive"]) for c in c5])
    md.run_batch(t, pats, qt, raw=True)
    torch.cuda.synchronize()
    # deep
    q64 = md.query64_tensor(0)
    r64 = torch.zeros(8, dtype=torch.int64, device="cuda")
    mp.launch_query_wide(t16, mp.Pattern.make("ring", 10), 0, False, q64.data_ptr(), r64.data_ptr(), 0, raw=True)
    torch.cuda.synchronize()
    print("done")


if __name__ == "__main__":
    main()
