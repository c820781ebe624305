#!/bin/bash
# quick parity + bench (pageable staging) + one sanitizer tool
mkdir -p gpurun_out
timeout 900 python -m pytest -q -x tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_scale.py > gpurun_out/pytest_quick.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_quick.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
python - <<'P'
import json
l=[x for x in open('gpurun_out/bench.log') if x.startswith('{')][-1]
d=json.loads(l)
print("pass", d["ms_per_step"], "e2e", d["e2e"]["ms_per_step"], d["e2e"]["ms_wall_all"], "pageable", d["e2e_pageable"])
print(sorted(d['kernels_ms'].items(), key=lambda kv:-kv[1])[:6])
P
bash tools/sanitize.sh ${1:-memcheck}
