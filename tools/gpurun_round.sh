#!/bin/bash
# one GPU session: tests, smoke, benches, launch list + one full ncu capture
#   CFGS="heat3d biharm"  bench these workloads
#   NCU_CFG=biharm KREGEX=biharm   profile this one (NCU=0 to skip)
set -u
mkdir -p gpurun_out
nvidia-smi > gpurun_out/smi.txt 2>&1
CFGS=${CFGS-heat3d}
NCU_CFG=${NCU_CFG:-heat3d}
KREGEX=${KREGEX:-$NCU_CFG}
if [ "${TESTS:-1}" = "1" ]; then
  timeout 1200 python -m pytest tests -m gpu -x -q ${PYTEST_K:-} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit=$?" >> gpurun_out/pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit=$?" >> gpurun_out/smoke.log
fi
for c in $CFGS; do
  timeout 900 python bench.py --config $c --steps ${STEPS:-5} --warmup 3 ${BENCH_ARGS:-} > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "bench exit=$?" >> gpurun_out/bench_$c.err
done
if [ "${NCU:-1}" = "1" ]; then
  C=$NCU_CFG
  timeout 600 python bench.py --config $C --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/plain.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$C.csv \
      python bench.py --config $C --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/ncu_launches.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$KREGEX -s ${SKIP:-3} -c 1 -o gpurun_out/prof_$C \
      python bench.py --config $C --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/ncu_full.log 2>&1
  echo "ncu exit=$?" >> gpurun_out/ncu_full.log
fi
