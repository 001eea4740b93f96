#!/bin/bash
# Dispatch chain breakdown: timer build of kx_dispatch, probe per config, then restore the normal build.
set -u
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
make -s NVFLAGS_EXTRA="-DKX_DISPATCH_TIMERS=1 ${EXTRA:-}" -B paper_2508_06948_b200/_lib/obj/kx_dispatch.o > gpurun_out/pd_build.log 2>&1 && make -s >> gpurun_out/pd_build.log 2>&1
for c in ${CONFIGS:-C4 C3 C2 C1}; do
  timeout 300 python scripts/dispatch_probe.py $c 3 > gpurun_out/pd_$c.log 2>&1; echo "probe rc=$?" >> gpurun_out/pd_$c.log
done
