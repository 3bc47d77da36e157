"""Hot-loop view of an ncu source capture (sass): per instruction, executions
and the warp-stall samples by reason.

  python scripts/ncu_sass_hot.py REP --kernel-index 0 --lo 0x5300 --hi 0x5d00
"""
import argparse
import collections
import csv
import io
import re
import subprocess

REASONS = ["stall_barrier", "stall_branch_resolving", "stall_dispatch", "stall_long_sb", "stall_math", "stall_mio",
           "stall_no_inst", "stall_not_selected", "stall_selected", "stall_short_sb", "stall_wait", "stall_misc"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--kernel-index", type=int, default=0)
    ap.add_argument("--lo", default="0")
    ap.add_argument("--hi", default="0xffffffff")
    ap.add_argument("--summary", action="store_true")
    a = ap.parse_args()
    out = subprocess.run(["ncu", "-i", a.rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    blocks = re.split(r'(?m)^"Kernel Name",', out)[1:]
    name, rest = blocks[a.kernel_index].split("\n", 1)
    rows = list(csv.reader(io.StringIO(rest)))
    hdr = rows[0]
    ie = hdr.index("Instructions Executed")
    rows = [r for r in rows[1:] if len(r) == len(hdr)]
    base = int(rows[0][0], 16)
    lo, hi = int(a.lo, 16), int(a.hi, 16)
    tot = collections.Counter()
    print(name[:100])
    for r in rows:
        off = int(r[0], 16) - base
        if not lo <= off < hi:
            continue
        st = {k: float(r[hdr.index(k)] or 0) for k in REASONS}
        for k, v in st.items():
            tot[k] += v
        tot["instr"] += float(r[ie] or 0)
        if not a.summary:
            top = sorted(st.items(), key=lambda kv: -kv[1])[:2]
            ts = " ".join(f"{k[6:]}={int(v)}" for k, v in top if v)
            print(f"{off:6x} {float(r[ie] or 0):10.0f}  {r[1].strip()[:60]:60s} {ts}")
    print("region totals:", dict(tot))


if __name__ == "__main__":
    main()
