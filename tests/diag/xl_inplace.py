"""One B200, one copy of the state: Hydro2D on a grid FOUR times BASELINE
configs[4] (65536 x 65536 cells, 137 GB of state) run in place
(config.aliases) -- the size 180 GB of HBM3e allows once the ping-pong copies
are gone.  Measurement / parity tool, not product code:

    python tests/diag/xl_inplace.py [N] [steps]      (default 65536, 2)

Prints one JSON line: the rate (CUDA events around lf_run) and whether full-width
row bands of the result equal the CPU oracle's bit for bit (the same check as
tests/test_gpu_hydro_large.py; the oracle import is the checker only)."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, str(__import__("pathlib").Path(__file__).resolve().parents[2]))
import oracle  # noqa: E402  (checker)
import paper_1710_08774_b200 as lf  # noqa: E402
from paper_1710_08774_b200 import inputs  # noqa: E402


def main():
    N = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    chunk = 1024
    free, total = torch.cuda.mem_get_info()
    need = 4 * (N + 4) ** 2 * 8
    if free < need * 1.06:
        raise SystemExit(f"needs {need / 1e9:.0f} GB of device memory, {free / 1e9:.0f} GB free")
    t0 = time.time()
    u = [torch.empty((N + 4, N + 4), dtype=torch.float64, device="cuda") for _ in range(4)]
    smax = 0.0
    for r0 in range(-2, N + 2, chunk):
        r1 = min(N + 2, r0 + chunk)
        rows, m = inputs.hydro_rows(N, N, r0, r1)
        smax = max(smax, m)
        for a, h in zip(u, rows):
            a[r0 + 2:r1 + 2].copy_(torch.from_numpy(h))
    dtdx = 0.5 / smax
    gen_s = time.time() - t0
    mass0 = [float(u[v][2:-2, 2:-2].sum()) for v in (0, 3)]
    plan = lf.Plan.with_ranges("hydro2d", (N, N), inplace=True)
    d = torch.tensor([dtdx], dtype=torch.float64, device="cuda")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    plan.run(u + [d] + u, steps=steps)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    peak = torch.cuda.max_memory_allocated()
    used = total - torch.cuda.mem_get_info()[0]
    ok = True
    bands = [(0, 24), (N // 2 - 12, N // 2 + 12), (N // 3, N // 3 + 24), (N - 24, N)]
    for a, b in bands:
        A, B = max(0, a - 2 * steps), min(N, b + 2 * steps)
        strip, _ = inputs.hydro_rows(N, N, A - 2, B + 2)
        ref = oracle.hydro(strip, dtdx, steps, fused=True)
        lo = a + 2 - (2 if a == 0 else 0)
        hi = b + 2 + (2 if b == N else 0)
        for v in range(4):
            got = u[v][lo:hi].cpu().numpy()
            ok &= bool(np.array_equal(got.view(np.uint64), ref[v][lo - A:hi - A].view(np.uint64)))
    cons = [abs(float(u[v][2:-2, 2:-2].sum()) - m0) / m0 for v, m0 in zip((0, 3), mass0)]
    print(json.dumps({"grid": [N, N], "steps": steps, "executor": plan.executor, "in_place": True,
                      "state_gb": round(need / 1e9, 1), "device_gb_in_use": round(used / 1e9, 1),
                      "torch_peak_gb": round(peak / 1e9, 1), "ms_per_step": round(ms / steps, 2),
                      "cell_steps_per_s": round(N * N * steps / (ms * 1e-3)), "row_bands_bit_exact": ok,
                      "bands": bands, "mass_energy_rel_drift": cons, "input_generation_s": round(gen_s, 1)}))
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
