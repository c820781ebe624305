#!/bin/bash
# Round profile bundle (run under gpurun): the gpu test suite, the full bench
# line (default run, with the reference CPU baseline), then an ncu launch list
# of one pass (device time + dram bytes per launch) and an ncu --set full
# capture of the dominant kernel.  Each ncu command follows a plain run of
# the same command that exited 0.
set -e
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -rA > gpurun_out/pytest_gpu.log 2>&1 || { tail -30 gpurun_out/pytest_gpu.log; exit 1; }
tail -1 gpurun_out/pytest_gpu.log
python bench.py > gpurun_out/bench_full.log 2>&1
tail -c 300 gpurun_out/bench_full.log
python tools/one_pass.py > gpurun_out/one_pass_plain.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv python tools/one_pass.py > gpurun_out/ncu_launch.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"${1:-k_mid_big}" -c 1 \
    -o gpurun_out/prof_dom -f python tools/one_pass.py > gpurun_out/ncu_full.log 2>&1
echo "profile bundle done"
