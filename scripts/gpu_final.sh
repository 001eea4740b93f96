#!/bin/bash
# Round evidence: smoke, all GPU tests, one bench line per config (with the
# CPU baseline and parity), ncu launch lists, full captures of the radix pass
# and of the phase-3 dispatch chain at C4.
set -u
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/f_smoke.log
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/f_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/f_pytest.log
for c in C4 C3 C2 C1; do
  timeout 600 python bench.py --config $c > gpurun_out/f_bench_$c.json 2> gpurun_out/f_bench_$c.err; echo "bench $c rc=$?" >> gpurun_out/f_bench_$c.err
done
timeout 600 python bench.py --impl reference > gpurun_out/f_ref.json 2> gpurun_out/f_ref.err
if [[ ${PROF:-1} == 1 ]]; then
  for c in C4 C3 C2 C1; do
    timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"^k_" --csv \
       --log-file gpurun_out/f_launches_$c.csv python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline \
       > /dev/null 2>&1
  done
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_onesweep_pass -s 5 -c 2 \
     -o gpurun_out/f_prof_onesweep -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_dispatch_chain -s 4 -c 1 \
     -o gpurun_out/f_prof_dispatch -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
fi
