#!/bin/bash
# VAR_ENV=LF_HEAT3D_VARIANT VARS="3 7 8 9" CFG=heat3d REPS=2 tools/tune_subset.sh
mkdir -p gpurun_out; : > gpurun_out/tune_${CFG}.txt
for rep in $(seq 1 ${REPS:-1}); do
for v in $VARS; do
  env $VAR_ENV=$v timeout 300 python bench.py --config $CFG --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/tune_${CFG}_$v.json 2>&1
  echo "variant $v $(python -c "import json;d=json.load(open('gpurun_out/tune_${CFG}_$v.json'));print(round(d['value']/1e9,2), round(d['ms_per_step'],3), round(d['roofline']['frac'],3), d['clocks']['reasons'])" 2>&1 | tail -1)" >> gpurun_out/tune_${CFG}.txt
done
done
