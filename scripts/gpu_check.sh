#!/bin/bash
# One GPU session: smoke, GPU parity tests, bench, ncu launch list + one full
# capture of the top kernel. Writes everything under gpurun_out/.
set -u
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
nproc > gpurun_out/nproc.txt; lscpu | grep -E "Model name|^CPU\(s\)" >> gpurun_out/nproc.txt
STAGE=${STAGE:-all}
if [[ $STAGE == all || $STAGE == tests ]]; then
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
  timeout 900 python -m pytest tests -q -m gpu -x ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
fi
if [[ $STAGE == all || $STAGE == bench ]]; then
  timeout 900 python bench.py --steps ${STEPS:-200} --warmup ${WARMUP:-5} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
fi
if [[ $STAGE == all || $STAGE == ncu ]]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"^k_" --csv \
     --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
     > gpurun_out/ncu_bench.log 2>&1; echo "ncu-list rc=$?" >> gpurun_out/ncu_bench.log
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${NCU_KERNEL:-k_onesweep_pass}" -s ${NCU_SKIP:-8} -c ${NCU_COUNT:-2} \
     -o gpurun_out/prof_top -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
     > gpurun_out/ncu_full.log 2>&1; echo "ncu-full rc=$?" >> gpurun_out/ncu_full.log
fi
