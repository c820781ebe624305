#!/bin/bash
# Round-end record (run under gpurun): gpu test suite, the reference arm and our
# default line as the driver runs them, our line for every other config, the
# multi-GPU estimate, then the ncu launch list (the full capture of the dominant kernel is a
# separate call: tools/ncu_kernels.sh k_mid_big -- one ncu per call).
mkdir -p gpurun_out/f
F=gpurun_out/f
python -m pytest tests -m gpu -q -rA > $F/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 $F/pytest_gpu.log
(time python bench.py --impl reference) > $F/ref_rmat22.log 2>&1; echo "ref rc=$?"
python bench.py > $F/ours_rmat22.log 2>&1; echo "ours rmat22 rc=$?"
for c in er1m ws4m chunglu ba2000; do
  python bench.py --config $c --steps 10 --warmup 3 > $F/ours_$c.log 2>&1; echo "ours $c rc=$?"
done
python tools/dist_estimate.py 2 4 8 > $F/dist_estimate.log 2>&1; echo "estimate rc=$?"
python tools/one_pass.py > $F/one_pass_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $F/launches.csv python tools/one_pass.py > $F/ncu_launch.log 2>&1; echo "launch list rc=$?"
