#!/bin/bash
# Replica sweeps (C5 shape) on one GPU: FCFS/oracle-T and Kairos/profiler-T,
# each with the reference Simulator timed on the host cores beside it.
set -u
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
R=${REPLICAS:-1024}
timeout 900 python scripts/replica_sweep.py --replicas $R --scheduler kairos --profile-T --cpu-sample 16 \
  > gpurun_out/sweep_kairos.json 2> gpurun_out/sweep_kairos.err; echo "rc=$?" >> gpurun_out/sweep_kairos.err
timeout 900 python scripts/replica_sweep.py --replicas $R --scheduler fcfs --cpu-sample 16 \
  > gpurun_out/sweep_fcfs.json 2> gpurun_out/sweep_fcfs.err; echo "rc=$?" >> gpurun_out/sweep_fcfs.err
if [[ ${NCU:-0} == 1 ]]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_replica_engine -c 1 \
    -o gpurun_out/prof_engine -f python scripts/replica_sweep.py --replicas 592 --duration 120 \
    --scheduler kairos --profile-T --cpu-sample 0 > gpurun_out/ncu_engine.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_engine.log
fi
