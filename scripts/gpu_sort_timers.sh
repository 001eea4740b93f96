#!/bin/bash
# Radix-pass tile phase breakdown in the C4 tick: rebuild with KX_SORT_TIMERS, run the probe.
set -u
mkdir -p gpurun_out
touch paper_2508_06948_b200/csrc/kx_order.cu paper_2508_06948_b200/csrc/kx_sortlib.cu
make NVFLAGS_EXTRA=-DKX_SORT_TIMERS=1 > gpurun_out/st_build.log 2>&1
timeout 300 python scripts/sort_timers.py > gpurun_out/st_probe.log 2>&1; echo "probe rc=$?" >> gpurun_out/st_probe.log
