#!/bin/bash
# Same-box A/B of several builds of the library (box-to-box variance is a few
# %, so compare builds inside one gpurun call).  Build each variant here and
# copy it to gpurun_ab/lib_<name>.so; then on the box:
#   NAMES="a b" bash tools/ab_libs.sh            (hydro bench line, 2 rounds)
#   NAMES="a b" CMD="python tools/rate_probe.py biharmonic2d 100 4096 4096" bash tools/ab_libs.sh
set -u
L=paper_1710_08774_b200/libloomfuse_b200.so
CMD=${CMD:-python bench.py --config hydro --steps 5 --warmup 3 --no-cpu --no-e2e}
cp $L /tmp/lib_keep.so
for r in 1 2; do
  for v in ${NAMES:-old new}; do
    cp gpurun_ab/lib_$v.so $L
    out=$($CMD 2>/dev/null | tail -1)
    echo "$v $(echo "$out" | python -c 'import json,sys
l=sys.stdin.read().strip()
try:
    d=json.loads(l); print("%.4g" % d["value"], "ms_per_step=%.3f" % d["ms_per_step"])
except Exception:
    print(l[-200:])')"
  done
done
cp /tmp/lib_keep.so $L
