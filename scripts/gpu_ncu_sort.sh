#!/bin/bash
# ncu --set full captures (with source) of the radix pass kernels in the C4 bench tick.
set -u
mkdir -p gpurun_out
for spec in ${SPECS:-old:2222:k_onesweep_pass new:4444:k_split_pass}; do
  name=${spec%%:*}; rest=${spec#*:}; rank=${rest%%:*}; kern=${rest#*:}
  KX_SORT_RANK=$rank timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$kern" -s ${SKIP:-5} -c 1 \
     -o gpurun_out/ncu_$name -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_$name.log 2>&1
  echo "rc=$?" >> gpurun_out/ncu_$name.log
done
