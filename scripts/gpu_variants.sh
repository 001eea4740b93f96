#!/bin/bash
# Dispatch-kernel A/B: rebuild kx_dispatch.cu with each NVX variant (timer build) and probe one config.
set -u
mkdir -p gpurun_out
: > gpurun_out/v_probe.log
IFS=';' read -ra VARS <<< "${VARIANTS:-}"
for v in "${VARS[@]}"; do
  make -s NVFLAGS_EXTRA="-DKX_DISPATCH_TIMERS=1 $v" -B paper_2508_06948_b200/_lib/obj/kx_dispatch.o > /dev/null 2>&1 && make -s > /dev/null 2>&1
  for c in ${CONFIGS:-C4}; do
    echo "=== $c [$v]" >> gpurun_out/v_probe.log
    timeout 300 python scripts/dispatch_probe.py $c 3 2>&1 | grep -E "dispatch |chain|cycles|decisions" >> gpurun_out/v_probe.log
  done
done
