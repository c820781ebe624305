#!/bin/bash
# A/B on the WS-4M and ER-1M configs (where the warp-per-seed kernels dominate): bench pass time + top kernels
for lib in "$@"; do
  for c in ws4m er1m; do
    EFG_LIB=$(realpath $lib) python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/abw.log 2>&1 || tail -5 gpurun_out/abw.log
    python - "$lib" "$c" <<'P'
import json, sys
l=[x for x in open('gpurun_out/abw.log') if x.startswith('{')][-1]
d=json.loads(l)
top=sorted(d['kernels_ms'].items(), key=lambda kv:-kv[1])[:4]
print(sys.argv[1].split('/')[-1], sys.argv[2], "pass", round(d['ms_per_step'],3), " ".join(f"{k}={v:.3f}" for k,v in top))
P
  done
done
