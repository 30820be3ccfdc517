#!/bin/bash
# Same-box A/B of two builds of the library (box-to-box variance is a few %,
# so compare builds inside one gpurun call).  Here: build each variant and copy
# it to gpurun_ab/lib_<name>.so; then on the box:
#   NAMES="old new" PROBE="hydro2d 20 4096 4096" bash tools/ab_libs.sh
set -u
L=paper_1710_08774_b200/libloomfuse_b200.so
cp $L /tmp/lib_keep.so
for r in 1 2; do
  for v in ${NAMES:-old new}; do
    cp gpurun_ab/lib_$v.so $L
    echo "$v $(python tools/rate_probe.py ${PROBE:-biharmonic2d 100 4096 4096} | sed 's/.*: //')"
  done
done
cp /tmp/lib_keep.so $L
