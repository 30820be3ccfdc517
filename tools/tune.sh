#!/bin/bash
# variant sweep: VAR_ENV=LF_BIHARM_VARIANT NVAR=6 CFG=biharm tools/tune.sh
mkdir -p gpurun_out
: > gpurun_out/tune_${CFG}.txt
for v in $(seq 0 $((NVAR-1))); do
  env $VAR_ENV=$v timeout 300 python bench.py --config $CFG --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/tune_${CFG}_$v.json 2>&1
  echo "variant $v $(python -c "import json;d=json.load(open('gpurun_out/tune_${CFG}_$v.json'));print(d['value']/1e9, d['ms_per_step'], round(d['roofline']['frac'],3))" 2>&1 | tail -1)" >> gpurun_out/tune_${CFG}.txt
done
