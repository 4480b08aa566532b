#!/bin/bash
# ncu --set full on a variant library: $1 tag, $2 lib, $3 variants
TAG=$1; LIB=$2; VARS=${3:-fused:0,seq}
mkdir -p gpurun_out
ODPO_LIB=$PWD/$LIB ncu --set full --clock-control none --import-source on -k regex:"k_engine|k_row_bwd" -c 6 \
    -o gpurun_out/${TAG}_prof -f python profiles/prof_kernels.py --config pythia --variants $VARS \
    > gpurun_out/${TAG}_prof.log 2>&1
tail -2 gpurun_out/${TAG}_prof.log
