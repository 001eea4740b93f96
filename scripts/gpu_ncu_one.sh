#!/bin/bash
# One ncu --set full capture (with source) of kernels matching $1 in the dispatch probe.
set -u
mkdir -p gpurun_out
K=${1:-k_dispatch_warp}; OUT=${2:-prof_one}; SKIP=${3:-2}; CNT=${4:-1}
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$K" -s $SKIP -c $CNT \
   -o gpurun_out/$OUT -f python scripts/dispatch_probe.py ${PER_POOL:-200000} 2 > gpurun_out/$OUT.log 2>&1; echo "rc=$?" >> gpurun_out/$OUT.log
