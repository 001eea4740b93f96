#!/bin/bash
# Dispatch-kernel cycle breakdown: rebuild with KX_DISPATCH_TIMERS, run the probe.
set -u
mkdir -p gpurun_out
touch paper_2508_06948_b200/csrc/kx_dispatch.cu
make NVFLAGS_EXTRA=-DKX_DISPATCH_TIMERS=1 > gpurun_out/t_build.log 2>&1
timeout 300 python scripts/dispatch_probe.py ${1:-2000000} 3 > gpurun_out/t_probe.log 2>&1; echo "probe rc=$?" >> gpurun_out/t_probe.log
