#!/bin/bash
# reference arm as the driver runs it + our default line + the other configs (ours)
mkdir -p gpurun_out/m2
R=gpurun_out/m2
(time python bench.py --impl reference) > $R/ref_rmat22.log 2>&1; echo "ref rmat22 rc=$?"
python bench.py > $R/ours_rmat22.log 2>&1; echo "ours rmat22 rc=$?"
for c in er1m ws4m chunglu ba2000; do
  python bench.py --config $c --steps 10 --warmup 3 > $R/ours_$c.log 2>&1; echo "ours $c rc=$?"
done
