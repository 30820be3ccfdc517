#!/bin/bash
# L2 promotion sweep: CFGS="box biharm heat3d" tools/promo.sh
mkdir -p gpurun_out; : > gpurun_out/promo.txt
for C in ${CFGS:-box biharm heat3d}; do
  for P in 0 64 128 256; do
    LF_TMA_PROMOTION=$P timeout 300 python bench.py --config $C --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/promo_tmp.json 2>&1
    echo "$C promo=$P $(python -c "import json;d=json.load(open('gpurun_out/promo_tmp.json'));print(round(d['value']/1e9,2), round(d['roofline']['frac'],3), d['clocks']['reasons'])" 2>&1 | tail -1)" >> gpurun_out/promo.txt
  done
done
