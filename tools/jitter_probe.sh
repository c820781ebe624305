# per-step device times of the default R-MAT22 line, several runs (host jitter inside timed steps)
for i in 1 2 3 4; do python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/j.log 2>&1; python -c "
import json; d=json.loads([x for x in open('gpurun_out/j.log') if x.startswith('{')][-1]); s=sorted(d['step_ms']); print(round(d['ms_per_step'],3), 'min', s[0], 'med', s[len(s)//2], 'max', s[-1])"; done
