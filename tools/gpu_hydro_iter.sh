#!/bin/bash
# one GPU iteration on the Hydro2D executor: parity tests, bench line, ncu
#   O=gpurun_out/<tag>  output dir; NCU=0 skips the profile; VARIANTS="0 1 2" sweeps LF_HYDRO_VARIANT
set -u
O=${O:-gpurun_out/hydro}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_hydro.py tests/test_gpu_fastmath.py tests/test_gpu_golden.py ${EXTRA_TESTS:-} -x -q > $O/pytest.log 2>&1; echo "exit=$?" >> $O/pytest.log
for v in ${VARIANTS:-1}; do
  LF_HYDRO_VARIANT=$v timeout 600 python bench.py --config hydro --steps 5 --warmup 3 --no-cpu --no-e2e > $O/bench_v$v.json 2> $O/bench_v$v.err
done
if [ "${NCU:-1}" = "1" ]; then
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:hydro_fused -s 3 -c 1 -o $O/prof_hydro \
     python bench.py --config hydro --steps 1 --warmup 1 --no-cpu --no-e2e > $O/ncu.log 2>&1; echo "ncu exit=$?" >> $O/ncu.log
fi
