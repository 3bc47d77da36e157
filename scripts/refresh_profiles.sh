#!/bin/bash
# One GPU-box pass that regenerates the round's measurement evidence into gpurun_out/
# (copied into profiles/ by hand after review):
#   bench lines (C4 headline + C1/C2/C3/C5 + the deep path), the ncu launch list of the
#   bench command, one `ncu --set full` capture of the three C4 kernels and of the deep
#   kernel, and the simulator report.
set -u
TAG=${1:-r01}
mkdir -p gpurun_out
python bench.py > gpurun_out/${TAG}_bench_c4_n1.json 2> gpurun_out/${TAG}_bench_c4.err
for c in c1 c2 c3 c5 deep; do
  python bench.py --config $c > gpurun_out/${TAG}_bench_$c.json 2> gpurun_out/${TAG}_bench_$c.err
done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_ncu_bench.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:esa_single -c 3 -o gpurun_out/${TAG}_full \
    python scripts/prof_one.py > gpurun_out/${TAG}_ncu_full.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:esa_deep -s 2 -c 2 -o gpurun_out/${TAG}_deep \
    python scripts/prof_deep.py > gpurun_out/${TAG}_ncu_deep.log 2>&1
python scripts/sim_report.py > gpurun_out/${TAG}_sim_report.json 2> gpurun_out/${TAG}_sim_report.err
tail -c 600 gpurun_out/${TAG}_bench_c4_n1.json
