#!/bin/bash
# biharm variant sweep (VARS="14 15 ...") after a bounded parity check of each
: > gpurun_out/bh_tests.txt
: > gpurun_out/tune_biharm.txt
for v in $VARS; do
  LF_BIHARM_VARIANT=$v timeout 120 python -m pytest tests/test_gpu_biharm.py -q -x > gpurun_out/pytest_bh_$v.log 2>&1
  echo "variant $v exit $? $(tail -1 gpurun_out/pytest_bh_$v.log)" >> gpurun_out/bh_tests.txt
  LF_BIHARM_VARIANT=$v timeout 120 python bench.py --config biharm --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/tune_biharm_$v.json 2>&1
  echo "variant $v $(python -c "import json;d=json.load(open('gpurun_out/tune_biharm_$v.json'));print(d['value']/1e9, d['ms_per_step'], round(d['roofline']['frac'],3))" 2>&1 | tail -1)" >> gpurun_out/tune_biharm.txt
done
