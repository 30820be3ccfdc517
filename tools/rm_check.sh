#!/bin/bash
# register-march check: generic-executor GPU tests, then box_jit / biharm_jit
# with the register march (default) and without it (LF_JIT_RM=0), same box
mkdir -p gpurun_out/rm
timeout 900 python -m pytest tests -m gpu -x -q -k "jit or golden or slabs" > gpurun_out/rm/pytest.log 2>&1; echo "pytest exit=$?" >> gpurun_out/rm/pytest.log
for c in ${CFGS:-box_jit biharm_jit}; do
  for rm in 1 0; do
    LF_JIT_RM=$rm timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu > gpurun_out/rm/bench_${c}_rm$rm.json 2> gpurun_out/rm/bench_${c}_rm$rm.err
  done
done
