#!/bin/bash
# One GPU iteration: gpu parity tests, then a short bench with the per-kernel table.
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
python bench.py --steps 10 --warmup 3 --no-cpu-baseline "$@" > gpurun_out/bench.log 2>&1 || tail -20 gpurun_out/bench.log
python - <<'P'
import json
l=[x for x in open('gpurun_out/bench.log') if x.startswith('{')][-1]
d=json.loads(l); print("ms_per_step", round(d['ms_per_step'],3), "e2e", d['e2e'])
for k,v in sorted(d['kernels_ms'].items(), key=lambda kv:-kv[1])[:12]: print(f"{v:8.3f} {k}")
P
