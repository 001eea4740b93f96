#!/bin/bash
# Replica-sweep scaling on one GPU (same per-replica load, C5 shape: 16
# instances, co-located workload at 12 workflows/s for 720 s per replica):
# 128/256/512/1024 replicas with clocks; the 1024 run also checks 4 sampled
# replicas bit-exact against the reference Simulator and times the 16-thread
# reference sample.
set -u
mkdir -p gpurun_out
: > gpurun_out/replica_scaling.jsonl
for r in ${SIZES:-128 256 512 1024}; do
  extra="--cpu-sample 0"
  if [ "$r" = "1024" ]; then extra="--cpu-sample 16 --parity 4"; fi
  timeout 900 python scripts/replica_sweep.py --replicas $r --duration 720 --rate 12 --instances 16 \
      --scheduler kairos --profile-T $extra >> gpurun_out/replica_scaling.jsonl 2> gpurun_out/replica_scaling_$r.err
  echo "replicas $r rc=$?"
done
