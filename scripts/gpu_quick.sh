#!/bin/bash
# Quick GPU iteration: GPU parity tests, dispatch probe, short bench (no CPU leg).
set -u
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests -q -m gpu -x ${PYTEST_ARGS:-} > gpurun_out/q_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/q_pytest.log
timeout 300 python scripts/dispatch_probe.py 2000000 3 > gpurun_out/q_probe.log 2>&1; echo "probe rc=$?" >> gpurun_out/q_probe.log
timeout 600 python bench.py --steps 200 --warmup 5 --no-cpu-baseline > gpurun_out/q_bench.json 2> gpurun_out/q_bench.err; echo "bench rc=$?" >> gpurun_out/q_bench.err
