#!/bin/bash
# A/B: CFG=heat3d tools/ab.sh  -> alternating runs with and without PDL
mkdir -p gpurun_out; : > gpurun_out/ab_${CFG}.txt
for rep in 1 2; do
  for mode in pdl nopdl; do
    if [ $mode = nopdl ]; then export LF_NO_PDL=1; else unset LF_NO_PDL; fi
    timeout 300 python bench.py --config $CFG --steps ${STEPS:-5} --warmup 3 --no-cpu --no-e2e > gpurun_out/ab_tmp.json 2>&1
    echo "$mode $(python -c "import json;d=json.load(open('gpurun_out/ab_tmp.json'));print(round(d['value']/1e9,2), round(d['ms_per_step'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'])" 2>&1 | tail -1)" >> gpurun_out/ab_${CFG}.txt
  done
done
