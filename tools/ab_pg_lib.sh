#!/bin/bash
# e2e from pageable host arrays across library builds: tools/ab_pg_lib.sh lib1.so lib2.so ...
mkdir -p gpurun_out
for rep in 1 2; do
  for lib in "$@"; do
    EFG_LIB=$(realpath $lib) python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 7 > gpurun_out/ab_pg.log 2>&1 || tail -5 gpurun_out/ab_pg.log
    python - "$lib" <<'P'
import json, sys
d = json.loads([x for x in open('gpurun_out/ab_pg.log') if x.startswith('{')][-1])
p = d['e2e_pageable']
print(sys.argv[1].split('/')[-1], "e2e", round(d['e2e']['ms_per_step'], 2), "pageable", round(p['ms_per_step'], 2), "h2d", round(p['ms_h2d'], 2), "all", p['ms_wall_all'])
P
  done
done
