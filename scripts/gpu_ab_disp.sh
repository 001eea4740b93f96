#!/bin/bash
# A/B of dispatch-kernel compile variants: parity tests, then the timer-build probe (C3, C4).
# VARIANTS="name1:-DFOO=1 name2:-DFOO=2,-DBAR=3"
set -u
mkdir -p gpurun_out
: > gpurun_out/abd.log
for spec in $VARIANTS; do
  name=${spec%%:*}; flags=${spec#*:}; flags=${flags//,/ }
  if [[ ${TESTS:-1} == 1 ]]; then
    make -s NVFLAGS_EXTRA="$flags" -B paper_2508_06948_b200/_lib/obj/kx_dispatch.o > gpurun_out/abd_build_$name.log 2>&1 && make -s >> gpurun_out/abd_build_$name.log 2>&1 || { echo "$name build failed" >> gpurun_out/abd.log; continue; }
    timeout 600 python -m pytest -q -x tests/test_gpu_dispatch.py tests/test_gpu_configs.py ${PYTEST_EXTRA:-} > gpurun_out/abd_t_$name.log 2>&1
    echo "$name tests rc=$? $(tail -1 gpurun_out/abd_t_$name.log)" >> gpurun_out/abd.log
  fi
  make -s NVFLAGS_EXTRA="-DKX_DISPATCH_TIMERS=1 $flags" -B paper_2508_06948_b200/_lib/obj/kx_dispatch.o > /dev/null 2>&1 && make -s > /dev/null 2>&1
  for c in ${CONFIGS:-C4 C3}; do
    timeout 300 python scripts/dispatch_probe.py $c 3 > gpurun_out/abd_p_${name}_$c.log 2>&1
    echo "$name $c: $(grep -A1 'no overlap' gpurun_out/abd_p_${name}_$c.log | head -0) $(grep '^dispatch ' gpurun_out/abd_p_${name}_$c.log) | $(grep 'us/record' gpurun_out/abd_p_${name}_$c.log | tail -1 | sed 's/.*loop/loop/') | $(grep 'resolver cycles' gpurun_out/abd_p_${name}_$c.log | tail -1 | sed 's/.*://')" >> gpurun_out/abd.log
  done
done
make -s -B paper_2508_06948_b200/_lib/obj/kx_dispatch.o > /dev/null 2>&1 && make -s > /dev/null 2>&1
