#!/bin/bash
# A/B of library builds on the GPU box: tools/ab.sh lib1.so lib2.so ... (bench pass time + top kernels each)
for rep in 1 2; do
  for lib in "$@"; do
    EFG_LIB=$(realpath $lib) python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ab.log 2>&1 || tail -5 gpurun_out/ab.log
    python - "$lib" <<'P'
import json, sys
l=[x for x in open('gpurun_out/ab.log') if x.startswith('{')][-1]
d=json.loads(l)
top=sorted(d['kernels_ms'].items(), key=lambda kv:-kv[1])[:4]
print(sys.argv[1].split('/')[-1], "pass", round(d['ms_per_step'],3), "e2e", round(d['e2e']['ms_per_step'],3), " ".join(f"{k}={v:.3f}" for k,v in top))
P
  done
done
