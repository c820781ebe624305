#!/bin/bash
# e2e from pageable host arrays against runtime settings: tools/ab_pageable.sh "" "EFG_STAGE_WORKERS=16" ...
mkdir -p gpurun_out
for rep in 1 2; do
  for cfg in "$@"; do
    env $cfg python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 6 > gpurun_out/ab_pg.log 2>&1 || tail -5 gpurun_out/ab_pg.log
    python - "$cfg" <<'P'
import json, sys
d = json.loads([x for x in open('gpurun_out/ab_pg.log') if x.startswith('{')][-1])
p = d['e2e_pageable']
print(repr(sys.argv[1]), "e2e", round(d['e2e']['ms_per_step'], 2), "pageable", round(p['ms_per_step'], 2), "h2d", round(p['ms_h2d'], 2), "all", p['ms_wall_all'])
P
  done
done
