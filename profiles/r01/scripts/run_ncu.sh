#!/bin/bash
# Profiling recipe (B200_PROFILING.md), run under gpurun from the repo root.
#   $1 = tag (output prefix), remaining args = extra bench.py flags
set -x
TAG=${1:-r01}; shift
mkdir -p gpurun_out
# 1) launch list with device times (cold-cache, serialised): shares, not absolutes
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${TAG}_launches.csv \
    python bench.py --steps 3 --warmup 1 --no-e2e --no-cpu "$@" > gpurun_out/${TAG}_launches_bench.log 2>&1
# 2) one full capture of the top kernels
ncu --set full --clock-control none --import-source on -k regex:"k_engine|k_row_bwd" -s 2 -c 2 \
    -o gpurun_out/${TAG}_prof -f \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu "$@" > gpurun_out/${TAG}_prof_bench.log 2>&1
ls -la gpurun_out
