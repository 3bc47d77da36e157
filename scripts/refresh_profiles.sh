#!/bin/bash
# One GPU-box pass that regenerates the round's measurement evidence into gpurun_out/
# (copied into profiles/ by hand after review):
#   bench lines (C4 headline + C1/C2/C3/C5 + the deep path), the ncu launch list of the
#   headline bench command, kernel-only probes (per-kernel times, strong-scaling shards,
#   three-stream overlap, deep-path rates) and the simulator report.
# The ncu --set full captures are separate (scripts/prof_configs.py + ncu_summary.py
# --configs, run on the box: the report itself exceeds gpurun's 64 MiB return limit).
set -u
TAG=${1:-r02}
# (the full ncu pass: ncu --set full --import-source on --clock-control none -k regex:esa_ \
#   -o gpurun_out/${TAG}_cfg python scripts/prof_configs.py, then ncu_summary.py --configs)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/${TAG}_smi.txt
python bench.py > gpurun_out/${TAG}_bench_c4_n1.json 2> gpurun_out/${TAG}_bench_c4.err
for c in c1 c2 c3 c5 deep; do
  python bench.py --config $c > gpurun_out/${TAG}_bench_$c.json 2> gpurun_out/${TAG}_bench_$c.err
done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-prune > gpurun_out/${TAG}_ncu_bench.log 2>&1
python scripts/kern_time.py > gpurun_out/${TAG}_kern_time.txt 2>&1
python scripts/shard_probe.py > gpurun_out/${TAG}_shard_probe.txt 2>&1
python scripts/stream_probe.py > gpurun_out/${TAG}_stream_probe.txt 2>&1
python scripts/graph_probe.py > gpurun_out/${TAG}_graph_probe.txt 2>&1
ncu --metrics gpu__time_duration.sum,sm__cycles_active.avg,launch__grid_size --clock-control none --csv \
    --log-file gpurun_out/${TAG}_fixed_cost.csv python scripts/fixed_probe.py > /dev/null 2>&1
python scripts/deep_rate.py > gpurun_out/${TAG}_deep_rate.txt 2>&1
python scripts/sim_report.py > gpurun_out/${TAG}_sim_report.json 2> gpurun_out/${TAG}_sim_report.err
tail -c 400 gpurun_out/${TAG}_bench_c4_n1.json
