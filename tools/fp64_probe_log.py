"""The fp64 roofline denominator with its clock record: tools/libfp64probe.so
(the DFMA-chain probe bench.py runs live for the Hydro2D roofline) read N
times with NVML SM-clock sampling around each reading.  Output: one JSON
object (profiles/r0N_fp64_probe.json).
usage: python tools/fp64_probe_log.py [readings]"""
import ctypes
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from bench import ClockSampler  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 5
    lib = ctypes.CDLL(str(ROOT / "tools" / "libfp64probe.so"))
    readings = []
    for _ in range(n):
        out = ctypes.c_double(0.0)
        with ClockSampler(0, period=0.005) as clk:
            if lib.lf_probe_fp64_tflops(5, ctypes.byref(out)) != 0:
                raise RuntimeError("fp64 probe failed")
        readings.append({"tflops": out.value, "clocks": clk.summary()})
    print(json.dumps({"probe": "tools/fp64_probe.cu (8 DFMA chains per thread, 8 CTAs of 256 per SM, best of 5)",
                      "readings": readings, "max_tflops": max(r["tflops"] for r in readings)}, indent=1))


if __name__ == "__main__":
    main()
