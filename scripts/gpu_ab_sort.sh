#!/bin/bash
# Radix-pass ranking variants (KX_SORT_RANK per pass) on the bench: launch lists.
set -u
for v in ${VARIANTS:-0000 1111 2222 0001 2221}; do
  KX_SORT_RANK=$v bash scripts/gpu_launches.sh; cp gpurun_out/launches.csv gpurun_out/launches_$v.csv
done
