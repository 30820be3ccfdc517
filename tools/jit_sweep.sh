#!/bin/bash
# sweep the generic executor's tile / prefetch / chunk knobs on one config
#   CFG=biharm_jit VARIANTS="TILE=1x512,PD=3 TILE=1x1024,PD=2" tools/jit_sweep.sh
set -u
mkdir -p gpurun_out
out=gpurun_out/jit_sweep_${CFG}.txt
: > $out
for v in $VARIANTS; do
  env_args=""
  for kv in ${v//,/ }; do env_args="$env_args LF_JIT_$kv"; done
  r=$(env $env_args timeout 300 python bench.py --config $CFG --steps 5 --warmup 3 --no-cpu --no-e2e 2>/dev/null | tail -1)
  echo "$v $(python -c "import json,sys; d=json.loads(sys.argv[1]); print(round(d['value']/1e9,2), round(d['roofline']['frac'],3))" "$r" 2>&1 | tail -1)" >> $out
done
