"""Pipe / issue summary of every kernel in an ncu report (raw page).

  python scripts/ncu_pipes.py gpurun_out/x.ncu-rep
"""
import csv
import io
import subprocess
import sys

WANT = ["gpu__time_duration.sum", "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "smsp__warps_eligible.avg.per_cycle_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "sm__cycles_elapsed.avg", "smsp__cycles_active.avg", "launch__registers_per_thread"]

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[0]
for r in rows[2:]:
    print(r[hdr.index("Kernel Name")][:70])
    print("   " + "  ".join(f"{w.split('.')[0].replace('sm__inst_executed_pipe_', '').replace('smsp__', '')}="
                            f"{r[hdr.index(w)]}" for w in WANT if w in hdr))
