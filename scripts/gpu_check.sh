#!/bin/bash
# Build locally and refuse to ship a stale library: used before every gpurun call.
set -e
cd "$(dirname "$0")/.."
make -s -j8 -C paper_2306_00606_b200 2>&1 | grep -E "error" && exit 1
for f in paper_2306_00606_b200/csrc/*.cu paper_2306_00606_b200/csrc/*.cuh include/efg.h; do
  if [ "$f" -nt paper_2306_00606_b200/libefg.so ]; then echo "STALE: $f newer than libefg.so"; exit 1; fi
done
make -s -C oracle
echo "build fresh"
