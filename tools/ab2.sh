#!/bin/bash
# A/B of library builds on the GPU box with a parity gate per build:
#   tools/ab2.sh lib1.so lib2.so ...
mkdir -p gpurun_out
for lib in "$@"; do
  EFG_LIB=$(realpath $lib) timeout 600 python -m pytest -q -x tests/test_gpu_parity.py \
     "tests/test_gpu_configs.py::test_rmat22_top_hubs_vs_oracle_fixtures" \
     "tests/test_gpu_configs.py::test_rmat22_engines_agree_on_every_seed" > gpurun_out/ab_parity.log 2>&1
  echo "$(basename $lib) parity: $(tail -1 gpurun_out/ab_parity.log)"
done
for rep in 1 2; do
  for lib in "$@"; do
    EFG_LIB=$(realpath $lib) python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/ab.log 2>&1 || tail -5 gpurun_out/ab.log
    python - "$lib" <<'P'
import json, sys
l=[x for x in open('gpurun_out/ab.log') if x.startswith('{')][-1]
d=json.loads(l)
top=sorted(d['kernels_ms'].items(), key=lambda kv:-kv[1])[:4]
print(sys.argv[1].split('/')[-1], "pass", round(d['ms_per_step'],3), "e2e", round(d['e2e']['ms_per_step'],3), " ".join(f"{k}={v:.3f}" for k,v in top))
P
  done
done
