#!/bin/bash
# one GPU session: tests, smoke, bench, launch list + one full ncu capture
set -u
mkdir -p gpurun_out
nvidia-smi > gpurun_out/smi.txt 2>&1
CFG=${CFG:-heat3d}
KREGEX=${KREGEX:-heat3d}
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py --config $CFG --steps 5 --warmup 3 > gpurun_out/bench_$CFG.json 2> gpurun_out/bench_$CFG.err; echo "bench exit=$?" >> gpurun_out/bench_$CFG.err
if [ "${NCU:-1}" = "1" ]; then
  timeout 600 python bench.py --config $CFG --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/plain.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$CFG.csv \
      python bench.py --config $CFG --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/ncu_launches.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$KREGEX -s 3 -c 1 -o gpurun_out/prof_$CFG \
      python bench.py --config $CFG --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/ncu_full.log 2>&1
  echo "ncu exit=$?" >> gpurun_out/ncu_full.log
fi
