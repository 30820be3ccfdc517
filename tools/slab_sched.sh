#!/bin/bash
# slab schedules side by side (tools/slab_probe.py per LF_SLAB_SCHEDULE)
O=${O:-gpurun_out/slab}; mkdir -p $O
for sch in default parallel whole concurrent; do
  echo "== $sch"
  for c in "heat3d 50 512 512 512" "heat3d 50 64 512 512" "biharmonic2d 100 512 4096" "hydro2d 10 4096 32768" "hydro2d 20 512 4096"; do
    if [ $sch = default ]; then timeout 600 python tools/slab_probe.py $c; else LF_SLAB_SCHEDULE=$sch timeout 600 python tools/slab_probe.py $c; fi
  done
done
