#!/bin/bash
# ncu launch list (per-kernel serialized device times) of a short bench run.
set -u
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"^k_" --csv \
   --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
   > gpurun_out/ncu_bench.log 2>&1; echo "ncu-list rc=$?" >> gpurun_out/ncu_bench.log
