set -u
mkdir -p gpurun_out
: > gpurun_out/abe.log
for v in base need1; do
  if [[ $v == need1 ]]; then export KX_TOPK_NEED=1; fi
  timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/abe_$v.json 2>/dev/null
  python - "$v" >> gpurun_out/abe.log <<'PY'
import json, sys
v = sys.argv[1]
d = json.loads(open(f"gpurun_out/abe_{v}.json").read().strip().splitlines()[-1])
print(v, "step %.3f ms" % d["ms_per_step"], " ".join("%s=%.3f" % (n, x["ms_per_step"]) for n, x in d["kernels"].items()))
PY
done
