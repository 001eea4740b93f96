#!/bin/bash
# A/B of runtime environment knobs on the C4 bench: VARIANTS="name:VAR=val,VAR2=val ..."
set -u
mkdir -p gpurun_out
: > gpurun_out/abe.log
for spec in $VARIANTS; do
  name=${spec%%:*}; envs=${spec#*:}; envs=${envs//,/ }
  env $envs timeout 300 python bench.py --config ${CONFIG:-C4} --steps ${STEPS:-100} --warmup 5 --no-cpu-baseline > gpurun_out/abe_$name.json 2>/dev/null
  python - "$name" >> gpurun_out/abe.log <<'PY'
import json, sys
v = sys.argv[1]
d = json.loads(open(f"gpurun_out/abe_{v}.json").read().strip().splitlines()[-1])
k = d["kernels"]
print(v, "step %.3f ms" % d["ms_per_step"], " ".join("%s=%.3f" % (n, x["ms_per_step"]) for n, x in k.items()))
PY
done
