#!/bin/bash
# register-march check: generic-executor GPU tests, then the 2D *_jit benches
# with each listed variant (VARIANTS="name:ENV=val,..."), same box
mkdir -p gpurun_out/rm
timeout 900 python -m pytest tests -m gpu -x -q -k "${PYK:-jit or golden or slabs or fastmath}" > gpurun_out/rm/pytest.log 2>&1; echo "pytest exit=$?" >> gpurun_out/rm/pytest.log
for c in ${CFGS:-box_jit biharm_jit}; do
  for v in ${VARIANTS:-base:X=1 norm:LF_JIT_RM=0}; do
    name=${v%%:*}; envs=${v#*:}
    env ${envs//,/ } timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu > gpurun_out/rm/bench_${c}_$name.json 2> gpurun_out/rm/bench_${c}_$name.err
  done
done
