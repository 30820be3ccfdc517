#!/bin/bash
# every bench workload once (bench lines for DESIGN.md's results table)
O=${O:-gpurun_out/benchall}; mkdir -p $O
nvidia-smi > $O/smi.txt 2>&1
timeout 1200 python bench.py --steps 3 --warmup 3 > $O/bench_hydro_large.json 2> $O/bench_hydro_large.err
for c in ${CFGS:-hydro hydro_large_adaptive hydro_inplace hydro_large_inplace heat3d biharm box heat3d_jit biharm_jit box_jit normalization_jit heat3d_jit_inplace biharm_jit_inplace}; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 > $O/bench_$c.json 2> $O/bench_$c.err
done
