#!/bin/bash
# C5 at full size: 1024 replicas x ~80K workflows (~256K requests) each,
# Kairos + profiler T, no CPU leg (the 16-replica CPU sample of
# gpu_sweep.sh gives the reference rate per request).
set -u
mkdir -p gpurun_out
free -g > gpurun_out/c5_mem.txt 2>&1; nproc >> gpurun_out/c5_mem.txt
timeout 1500 python scripts/replica_sweep.py --replicas 1024 --duration ${DURATION:-6700} --scheduler kairos --profile-T \
  --cpu-sample 0 > gpurun_out/sweep_c5_kairos.json 2> gpurun_out/sweep_c5_kairos.err; echo "rc=$?" >> gpurun_out/sweep_c5_kairos.err
