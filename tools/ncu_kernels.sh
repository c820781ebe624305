#!/bin/bash
# ncu --set full of several kernels of one R-MAT22 pass (one capture each), after a plain run
mkdir -p gpurun_out
python tools/one_pass.py > gpurun_out/one_pass_plain.log 2>&1 || exit 1
for k in "$@"; do
  ncu --set full --import-source on --clock-control none -k regex:"$k" -c 1 -o gpurun_out/k_$k -f \
      python tools/one_pass.py > gpurun_out/ncu_$k.log 2>&1; echo "$k rc=$?"
done
