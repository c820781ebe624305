#!/bin/bash
# e2e (pinned host inputs) against the staging split: tools/ab_stage.sh "25" "10,25,45" ...  (cumulative % of 2m)
mkdir -p gpurun_out
for rep in 1 2; do
  for cfg in "$@"; do
    EFG_STAGE_SPLITS=$cfg python bench.py --config ${CONFIG:-rmat22} --steps 3 --warmup 3 --no-cpu-baseline \
      --e2e-steps 10 > gpurun_out/ab_stage.log 2>&1 || tail -5 gpurun_out/ab_stage.log
    python - "$cfg" <<'P'
import json, sys
d = json.loads([x for x in open('gpurun_out/ab_stage.log') if x.startswith('{')][-1])
e, p = d['e2e'], d['e2e_pageable']
print(sys.argv[1], "pass", round(d['ms_per_step'], 2), "e2e", round(e['ms_per_step'], 2), "dev", round(e['ms_device_events'], 2),
      "prep", round(e['ms_prepare'], 2), "h2d", round(e['ms_h2d'], 2), "pageable", round(p['ms_per_step'], 2), "all", e['ms_wall_all'])
P
  done
done
