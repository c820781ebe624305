#!/bin/bash
# A/B of library builds (EFG_LIB) with the parity gate, printing chosen kernels' live times:
#   KERNELS="k_hist_block k_hist_count" tools/ab_kern.sh lib1.so lib2.so ...
mkdir -p gpurun_out
for lib in "$@"; do
  EFG_LIB=$(realpath $lib) timeout 600 python -m pytest -q -x tests/test_gpu_parity.py \
     "tests/test_gpu_configs.py::test_rmat22_top_hubs_vs_oracle_fixtures" > gpurun_out/abk_parity.log 2>&1
  echo "$(basename $lib) parity: $(tail -1 gpurun_out/abk_parity.log)"
done
for rep in 1 2; do
  for lib in "$@"; do
    EFG_LIB=$(realpath $lib) python bench.py --config ${CONFIG:-rmat22} --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/abk.log 2>&1 || tail -5 gpurun_out/abk.log
    python - "$lib" "$KERNELS" <<'P'
import json, sys
d = json.loads([x for x in open('gpurun_out/abk.log') if x.startswith('{')][-1])
want = sys.argv[2].split()
ks = {k: v for k, v in d['kernels_ms'].items() if any(w in k for w in want)}
print(sys.argv[1].split('/')[-1], "pass", round(d['ms_per_step'], 3), "e2e", round(d['e2e']['ms_per_step'], 3),
      " ".join(f"{k}={v:.3f}" for k, v in sorted(ks.items())))
P
  done
done
