#!/bin/bash
TAG=${1:-r01b}; CFG=${2:-pythia}; VARS=${3:-fused:0,fused:3,two_pass:0,seq}
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:"k_engine|k_row_bwd" -c 10 \
    -o gpurun_out/${TAG}_prof -f python profiles/prof_kernels.py --config $CFG --variants $VARS \
    > gpurun_out/${TAG}_prof.log 2>&1
tail -3 gpurun_out/${TAG}_prof.log
