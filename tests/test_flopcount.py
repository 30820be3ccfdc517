"""The Hydro2D flop count bench.py divides by (oracle/flopcount.cpp)."""
import json
import subprocess

import bench
import oracle


def test_hydro_flops_per_cell_step_matches_the_count():
    subprocess.run(["make", "-s", "-C", str(oracle.DIR), "flopcount"], check=True)
    exe = oracle.DIR / "flopcount"
    d = json.loads(subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout)
    assert abs(d["flops_per_cell_step"] - bench.HYDRO_FLOPS_PER_CELL_STEP) < 1e-3
    # 10 Newton steps of 2 sqrt + 1 division dominate (fma = 2 flops): O(10^3) per cell-step
    per = d["per_cell_sweep"]
    assert per["sqrt"] == 26 and per["div"] == 18  # quotients as reciprocal x numerator
