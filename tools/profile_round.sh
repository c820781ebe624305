#!/bin/bash
# Round profile bundle (run under gpurun): full bench line, ncu launch list with
# dram bytes of one pass, and an ncu --set full capture of the dominant kernel.
set -e
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_full.log 2>&1
python tools/one_pass.py > /dev/null
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv python tools/one_pass.py > gpurun_out/ncu_launch.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"${1:-k_mid_block}" -c 1 \
    -o gpurun_out/prof_dom python tools/one_pass.py > gpurun_out/ncu_full.log 2>&1
tail -c 400 gpurun_out/bench_full.log
