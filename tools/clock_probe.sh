# per-step device times of short configs (host jitter inside timed steps): bash tools/clock_probe.sh
for c in ws4m er1m; do for i in 1 2 3 4 5; do python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/w.log 2>&1; python -c "
import json; d=json.loads([x for x in open('gpurun_out/w.log') if x.startswith('{')][-1]); s=d['step_ms']; print('$c', round(d['ms_per_step'],2), 'max', max(s), 'samples', d['clocks']['samples'])"; done; done
