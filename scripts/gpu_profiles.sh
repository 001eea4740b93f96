#!/bin/bash
# Round profiles: ncu launch list of each bench config, one --set full capture
# of the radix pass and of the dispatch chain kernel at C4.
set -u
mkdir -p gpurun_out
for c in ${CONFIGS:-C4 C3 C2 C1}; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"^k_" --csv \
     --log-file gpurun_out/launches_$c.csv python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline \
     > gpurun_out/ncu_bench_$c.log 2>&1; echo "ncu-list rc=$?" >> gpurun_out/ncu_bench_$c.log
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_onesweep_pass -s 5 -c 2 \
   -o gpurun_out/prof_onesweep -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full_sort.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_dispatch_chain -s 3 -c 1 \
   -o gpurun_out/prof_dispatch -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full_disp.log 2>&1
