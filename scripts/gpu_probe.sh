#!/bin/bash
# Dispatch-kernel iteration: dispatch/config parity tests, then a timer build and probes of C4 and C3.
set -u
mkdir -p gpurun_out
timeout 600 python -m pytest -q -x tests/test_gpu_dispatch.py tests/test_gpu_configs.py ${PYTEST_EXTRA:-} > gpurun_out/p_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/p_pytest.log
make -s NVFLAGS_EXTRA="-DKX_DISPATCH_TIMERS=1 ${NVX:-}" -B paper_2508_06948_b200/_lib/obj/kx_dispatch.o > /dev/null 2>&1 && make -s > /dev/null 2>&1
for c in ${CONFIGS:-C4 C3}; do
  timeout 300 python scripts/dispatch_probe.py $c 3 > gpurun_out/p_probe_$c.log 2>&1; echo "probe rc=$?" >> gpurun_out/p_probe_$c.log
done
