#!/bin/bash
# Build libefg.so with extra nvcc flags into paper_2306_00606_b200/variants/<name>.so (A/B on the GPU with tools/ab.sh).
# usage: tools/build_variant.sh NAME "-DFOO=1 -DBAR=2"
set -e
cd "$(dirname "$0")/.."
name=$1; flags=$2
B=/tmp/efg_variant_$name
rm -rf $B; mkdir -p $B/pkg paper_2306_00606_b200/variants
cp -r include $B/include
cp -r paper_2306_00606_b200/csrc paper_2306_00606_b200/Makefile $B/pkg/
make -s -j8 -C $B/pkg EXTRA_NVFLAGS="$flags" > /dev/null
cp $B/pkg/libefg.so paper_2306_00606_b200/variants/$name.so
echo "built variants/$name.so ($flags)"
