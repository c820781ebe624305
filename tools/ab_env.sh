#!/bin/bash
# A/B of runtime settings (environment assignments) on the in-tree library:
#   tools/ab_env.sh "" "EFG_X=1" "EFG_X=2 EFG_Y=3" ...
mkdir -p gpurun_out
for rep in 1 2; do
  for cfg in "$@"; do
    env $cfg python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/ab_env.log 2>&1 || tail -5 gpurun_out/ab_env.log
    python - "$cfg" <<'P'
import json, sys
d = json.loads([x for x in open('gpurun_out/ab_env.log') if x.startswith('{')][-1])
top = sorted(d['kernels_ms'].items(), key=lambda kv: -kv[1])[:4]
print(repr(sys.argv[1]), "pass", round(d['ms_per_step'], 3), "e2e", round(d['e2e']['ms_per_step'], 3),
      " ".join(f"{k}={v:.3f}" for k, v in top))
P
  done
done
grep -h '\[efg\]' gpurun_out/ab_env.log | head -2
