#!/bin/bash
# ncu launch list + one --set full capture per config (one gpurun call)
#   CFGS="heat3d biharm box hydro" tools/profile_all.sh
mkdir -p gpurun_out
for C in ${CFGS:-heat3d biharm box hydro}; do
  case $C in heat3d) K=heat3d;; biharm) K=biharm;; box) K=box_fused;; hydro*) K=hydro_fused;; *_jit*) K=lf_jit_step;; *) K=$C;; esac
  SKIP=3; case $C in box|box_jit) SKIP=1;; esac
  timeout 600 python bench.py --config $C --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/plain_$C.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$C.csv \
      python bench.py --config $C --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/ncu_launches_$C.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s $SKIP -c 1 -o gpurun_out/prof_$C \
      python bench.py --config $C --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/ncu_full_$C.log 2>&1
  echo "$C ncu exit=$?" >> gpurun_out/profile_all.log
done
