#!/bin/bash
# Quick GPU iteration: GPU parity tests, dispatch probes (timer build), short bench (no CPU leg).
set -u
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -q -m gpu -x ${PYTEST_ARGS:-} > gpurun_out/q_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/q_pytest.log
for c in ${CONFIGS:-C4 C3}; do
  timeout 400 python bench.py --config $c --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/q_bench_$c.json 2> gpurun_out/q_bench_$c.err; echo "bench $c rc=$?" >> gpurun_out/q_bench_$c.err
done
make -s NVFLAGS_EXTRA=-DKX_DISPATCH_TIMERS=1 -B paper_2508_06948_b200/_lib/obj/kx_dispatch.o > /dev/null 2>&1 && make -s > /dev/null 2>&1
for c in ${CONFIGS:-C4 C3}; do
  timeout 300 python scripts/dispatch_probe.py $c 3 > gpurun_out/q_probe_$c.log 2>&1; echo "probe rc=$?" >> gpurun_out/q_probe_$c.log
done
