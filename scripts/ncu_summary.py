"""Summarise ncu outputs brought back in gpurun_out/ into profiles/ (tracked).

  python scripts/ncu_summary.py --rep gpurun_out/prof.ncu-rep --launches gpurun_out/launches.csv --tag r01
"""
import argparse
import csv
import io
import json
import os
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg", "smsp__inst_executed.sum",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__inst_issued.avg.pct_of_peak_sustained_active",
    "sm__instruction_throughput.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_adu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_cbu.avg.pct_of_peak_sustained_active",
    "smsp__thread_inst_executed_per_inst_executed.ratio", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
]
STALLS = ["smsp__pcsamp_warps_issue_stalled_" + s for s in (
    "wait", "short_scoreboard", "long_scoreboard", "math_pipe_throttle", "mio_throttle", "not_selected",
    "selected", "branch_resolving", "barrier", "dispatch_stall", "no_instructions", "lg_throttle", "membar")]


def raw_rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")]}
        for m in METRICS + STALLS:
            if m in hdr:
                v = r[hdr.index(m)]
                try:
                    d[m] = float(v.replace(",", ""))
                except ValueError:
                    d[m] = v
                d[m + ".unit"] = units[hdr.index(m)]
        res.append(d)
    return res


def _bytes(v, unit):
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Kibyte": 1024, "Mibyte": 1 << 20}.get(unit, 1)


def _us(v, unit):
    return v / 1e3 if unit in ("nsecond", "ns") else (v * 1e3 if unit in ("msecond", "ms") else v)


def launches(path):
    rows = [r for r in csv.reader(open(path)) if r]
    i = next(k for k, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[i]
    agg = {}
    for r in rows[i + 1:]:
        if len(r) != len(hdr) or r[hdr.index("Metric Name")] != "gpu__time_duration.sum":
            continue
        name = r[hdr.index("Kernel Name")]
        unit = r[hdr.index("Metric Unit")]
        v = float(r[hdr.index("Metric Value")].replace(",", ""))
        v_us = v / 1e3 if unit in ("nsecond", "ns") else (v * 1e3 if unit in ("msecond", "ms") else v)
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v_us
    tot = sum(v[1] for v in agg.values())
    return [{"kernel": k, "launches": n, "total_us": t, "mean_us": t / n, "share": t / tot}
            for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep")
    ap.add_argument("--launches")
    ap.add_argument("--tag", required=True)
    ap.add_argument("--configs", action="store_true",
                    help="the report is scripts/prof_configs.py's: also write profiles/ncu_summary.json "
                         "(per-launch DRAM bytes and C4 lane-instructions per embedding)")
    a = ap.parse_args()
    out = {"tag": a.tag}
    if a.rep:
        out["full"] = raw_rows(a.rep)
        if a.configs:
            sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
            from prof_configs import KERNELS  # noqa: E402  (index -> config)
            full = [k for k in out["full"] if "esa_" in k["kernel"]]
            assert len(full) == len(KERNELS), (len(full), len(KERNELS))
            byk = dict(zip(KERNELS, full))
            dram = {n: _bytes(k["dram__bytes_read.sum"], k["dram__bytes_read.sum.unit"]) +
                    _bytes(k["dram__bytes_write.sum"], k["dram__bytes_write.sum.unit"]) for n, k in byk.items()}
            emb = 652458240  # P(32,6): one C4 RAW launch
            summ = {"source": f"profiles/{a.tag}_ncu.json (ncu --set full, scripts/prof_configs.py: one launch of "
                              f"each config's dominant kernel)",
                    "dram_bytes_per_launch": {n[3:]: dram[n] for n in KERNELS[:3]},
                    "lane_instr_per_embedding": {n[3:]: byk[n]["smsp__inst_executed.sum"] * 32 / emb
                                                 for n in KERNELS[:3]},
                    # shared-memory data-pipe wavefronts (1 per SM per clock at most) per embedding
                    "smem_wavefronts_per_embedding": {
                        n[3:]: byk[n]["l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"] / emb for n in KERNELS[:3]},
                    "kernel_us_ncu": {n: _us(byk[n]["gpu__time_duration.sum"], byk[n]["gpu__time_duration.sum.unit"])
                                      for n in KERNELS},
                    "config_traffic": {n: dram[n] for n in KERNELS[3:]}}
            summ["config_traffic"]["c4"] = dram["c4_preserve_sensitive"]
            with open("profiles/ncu_summary.json", "w") as f:
                json.dump(summ, f, indent=1)
    if a.launches:
        out["launch_list"] = launches(a.launches)
    os.makedirs("profiles", exist_ok=True)
    with open(f"profiles/{a.tag}_ncu.json", "w") as f:
        json.dump(out, f, indent=1)
    for k in out.get("full", []):
        print(k["kernel"][:70])
        for m in METRICS + STALLS:
            if m in k:
                print(f"   {m} = {k[m]} {k.get(m + '.unit', '')}")
    for l in out.get("launch_list", []):
        print(f"{l['share']*100:6.2f}%  {l['launches']:4d} x {l['mean_us']:10.1f} us  {l['kernel'][:90]}")


if __name__ == "__main__":
    sys.exit(main())
