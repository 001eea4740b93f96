#!/bin/bash
# A/B of engine build variants on a replica sweep (no CPU leg).
# VARIANTS="name1:-DFOO=1 name2:-DFOO=2"
set -u
mkdir -p gpurun_out
: > gpurun_out/abe.log
for spec in $VARIANTS; do
  name=${spec%%:*}; flags=${spec#*:}; flags=${flags//,/ }
  touch paper_2508_06948_b200/csrc/kx_engine.cu
  make NVFLAGS_EXTRA="$flags" > gpurun_out/abe_build_$name.log 2>&1 || { echo "$name build failed" >> gpurun_out/abe.log; continue; }
  for sch in kairos fcfs; do
    extra=""; [[ $sch == kairos ]] && extra="--profile-T"
    timeout 600 python scripts/replica_sweep.py --replicas ${REPLICAS:-1024} --duration ${DURATION:-360} \
      --scheduler $sch $extra --cpu-sample 0 > gpurun_out/abe_${name}_$sch.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/abe_${name}_$sch.json'));print('$name', '$sch', round(d['device_ms'],1), 'ms', round(d['value']))" >> gpurun_out/abe.log
  done
done
