set -u
O=gpurun_out/r2b; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_jit.py -q -k fault > $O/pytest_fault.log 2>&1; echo "exit=$?" >> $O/pytest_fault.log
timeout 900 python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > $O/plain.json 2> $O/plain.err && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_hydro_large.csv \
      python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > $O/ncu_launches.log 2>&1
echo "launches exit=$?" >> $O/ncu_launches.log
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:hydro_fused -s 2 -c 1 -o $O/prof_hydro_large \
      python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > $O/ncu_full.log 2>&1
echo "ncu exit=$?" >> $O/ncu_full.log
