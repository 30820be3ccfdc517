"""The device's exact-division sequence for x/3.0f (lf_div3f) is bit-identical
to IEEE division for every float -- checked exhaustively over all 2^32 bit
patterns by oracle/div3check (C, OpenMP)."""
import json
import subprocess

import oracle


def test_div3_sequence_exhaustive():
    subprocess.run(["make", "-s", "-C", str(oracle.DIR), "div3check"], check=True)
    r = subprocess.run([str(oracle.DIR / "div3check")], capture_output=True, text=True, timeout=600)
    d = json.loads(r.stdout)
    assert d["checked"] == 2 ** 32 and d["mismatches"] == 0
