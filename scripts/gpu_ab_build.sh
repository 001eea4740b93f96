#!/bin/bash
# A/B of compile-time variants (NVFLAGS_EXTRA per variant) on the bench.
# VARIANTS="name1:-DFOO=1 name2:-DFOO=2"
set -u
mkdir -p gpurun_out
: > gpurun_out/abb.log
for spec in $VARIANTS; do
  name=${spec%%:*}; flags=${spec#*:}; flags=${flags//,/ }
  touch ${TOUCH:-paper_2508_06948_b200/csrc/*.cu}
  make NVFLAGS_EXTRA="$flags" > gpurun_out/abb_build_$name.log 2>&1 || { echo "$name build failed" >> gpurun_out/abb.log; continue; }
  if [[ ${TESTS:-1} == 1 ]]; then
    timeout 300 python -m pytest tests/test_gpu_order.py tests/test_gpu_dispatch.py -q -x > gpurun_out/abb_t_$name.log 2>&1
    echo "$name tests rc=$? $(tail -1 gpurun_out/abb_t_$name.log)" >> gpurun_out/abb.log
  fi
  timeout 300 python bench.py --steps ${STEPS:-100} --warmup 5 --no-cpu-baseline > gpurun_out/abb_$name.json 2>/dev/null
  python - "$name" >> gpurun_out/abb.log <<'PY'
import json, sys
v = sys.argv[1]
d = json.loads(open(f"gpurun_out/abb_{v}.json").read().strip().splitlines()[-1])
k = d["kernels"]
print(v, "step %.3f ms" % d["ms_per_step"], " ".join("%s=%.3f" % (n, x["ms_per_step"]) for n, x in k.items()))
PY
done
