#!/bin/bash
# Round measurement of record (run under gpurun): the reference arm as the
# driver runs it, its stratified extrapolation, and our bench line for every
# BASELINE config (each with the reference CPU baseline beside it), plus the
# reference's full-graph runs for the configs where those take seconds.
mkdir -p gpurun_out/m
R=gpurun_out/m
python bench.py --impl reference --steps 20 --warmup 3 > $R/ref_rmat22.log 2>&1; echo "ref rmat22 rc=$?"
python bench.py --impl reference --steps 1 --warmup 0 --ref-stratified > $R/ref_rmat22_strat.log 2>&1; echo "ref strat rc=$?"
python bench.py --cpu-port > $R/ours_rmat22_port.log 2>&1; echo "ours rmat22 rc=$?"
for c in er1m ws4m chunglu ba2000; do
  python bench.py --config $c --steps 10 --warmup 3 > $R/ours_$c.log 2>&1; echo "ours $c rc=$?"
done
for c in ba2000 er1m ws4m; do
  python bench.py --impl reference --config $c --steps 1 --warmup 0 > $R/ref_$c.log 2>&1; echo "ref $c rc=$?"
done
python bench.py --impl reference --config chunglu --steps 3 --warmup 1 --ref-stratified > $R/ref_chunglu.log 2>&1; echo "ref chunglu rc=$?"
