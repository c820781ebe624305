#!/bin/bash
# ncu --set full of k_mid_big for each given library (EFG_LIB), one pass of R-MAT22 each
mkdir -p gpurun_out
for lib in "$@"; do
  name=$(basename $lib .so)
  EFG_LIB=$(realpath $lib) python tools/one_pass.py > gpurun_out/plain_$name.log 2>&1 && \
  EFG_LIB=$(realpath $lib) ncu --set full --import-source on --clock-control none -k regex:k_mid_big -c 1 \
      -o gpurun_out/mid_$name -f python tools/one_pass.py > gpurun_out/ncu_$name.log 2>&1
  echo "$name rc=$?"
done
