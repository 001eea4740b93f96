#!/bin/bash
# A/B of radix-pass ranking variants (KX_SORT_RANK per pass) on the bench
# (per-kernel times from direct launches) + order parity tests per variant.
set -u
mkdir -p gpurun_out
: > gpurun_out/ab.log
for v in ${VARIANTS:-2221 3333 3331}; do
  KX_SORT_RANK=$v timeout 300 python -m pytest tests/test_gpu_order.py -q -x > gpurun_out/ab_t_$v.log 2>&1
  echo "$v tests rc=$? $(tail -1 gpurun_out/ab_t_$v.log)" >> gpurun_out/ab.log
  KX_SORT_RANK=$v timeout 300 python bench.py --steps ${STEPS:-100} --warmup 5 --no-cpu-baseline > gpurun_out/ab_$v.json 2>/dev/null
  python - "$v" >> gpurun_out/ab.log <<'PY'
import json, sys
v = sys.argv[1]
d = json.loads(open(f"gpurun_out/ab_{v}.json").read().strip().splitlines()[-1])
k = d["kernels"]
print(v, "step %.3f ms" % d["ms_per_step"], " ".join("%s=%.3f" % (n, x["ms_per_step"]) for n, x in k.items()))
PY
done
