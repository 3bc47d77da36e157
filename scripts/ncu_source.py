"""Per-source-line instruction / stall attribution from an ncu report captured
with --import-source on (kernels compiled with -lineinfo).

  python scripts/ncu_source.py gpurun_out/x.ncu-rep [--kernel REGEX] [--top 30]
"""
import argparse
import csv
import io
import re
import subprocess


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--kernel", default="esa_single")
    ap.add_argument("--top", type=int, default=30)
    ap.add_argument("--view", default="cuda")
    a = ap.parse_args()
    out = subprocess.run(["ncu", "-i", a.rep, "--page", "source", "--csv", "--print-source", a.view],
                         capture_output=True, text=True).stdout
    blocks = re.split(r'(?m)^"Kernel Name",', out)
    for blk in blocks[1:]:
        name, rest = blk.split("\n", 1)
        if not re.search(a.kernel, name):
            continue
        rows = list(csv.reader(io.StringIO(rest)))
        hdr = rows[0]
        ie = hdr.index("Instructions Executed")
        ss = hdr.index("Warp Stall Sampling (All Samples)")
        src = hdr.index("Source")
        loc = hdr.index("# Address") if "# Address" in hdr else (hdr.index("Line") if "Line" in hdr else 0)
        data = []
        for r in rows[1:]:
            if len(r) != len(hdr):
                continue
            try:
                n = float(r[ie] or 0)
                s = float(r[ss] or 0)
            except ValueError:
                continue
            data.append((n, s, r[loc], r[src].strip()[:110]))
        tot = sum(d[0] for d in data) or 1
        tots = sum(d[1] for d in data) or 1
        print(f"== {name.strip()[:120]}\n   total warp instrs {tot:.4g}, stall samples {tots:.4g}")
        for n, s, l, t in sorted(data, key=lambda d: -d[0])[:a.top]:
            print(f"  {100 * n / tot:5.1f}% instr {100 * s / tots:5.1f}% samp  L{l:>5}  {t}")


if __name__ == "__main__":
    main()
