#!/usr/bin/env python
"""Benchmark of the fused stencil-chain path (BASELINE.json metric:
fused-chain cell-updates/s, % of HBM roofline, vs host CPU).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl loomfuse|reference]
                    [--config heat3d|biharm|box|hydro|hydro_large]

A bench "step" is one full run of the configured chain over its grid (e.g.
configs[1]: 50 time steps of the 3D heat chain on 512^3).  N=1 is the default;
for N>1 launch under torchrun (one rank per GPU, NCCL): the outer dimension is
split into slabs and faces are exchanged every time step (strong scaling, the
grid is fixed).  Rank 0 prints one JSON line.

--impl reference times the reference's CPU path -- the HFAV-style fused CPU
schedule restated in oracle/ (the reference's own executor is absent from the
snapshot) -- on all host threads, on a bounded sample.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

FALLBACK_HBM_GBS = 6650.0


# --------------------------------------------------------------------- workloads
def _heat3d_inputs(sizes, seed=0):
    from paper_1710_08774_b200 import inputs
    return [inputs.heat3d_input(*sizes, seed=seed)]


def _biharm_inputs(sizes, seed=0):
    from paper_1710_08774_b200 import inputs
    return [inputs.biharm_input(*sizes, seed=seed)]


def _box_inputs(sizes, seed=0):
    from paper_1710_08774_b200 import inputs
    return [inputs.box_input(*sizes, seed=seed)]


def _norm_inputs(sizes, seed=0):
    rng = np.random.default_rng(seed)
    return [rng.random((sizes[0], sizes[1] + 1)), np.zeros(sizes[0])]


def _hydro_inputs(sizes, seed=0):
    from paper_1710_08774_b200 import inputs
    st, dtdx = inputs.hydro_input(*sizes, seed=seed)
    return st + [np.array([dtdx], dtype=np.float64)]


# slab generators: the axioms of one rank's slab [lo, hi) of the outer
# dimension (storage rows incl. halo), built without the whole grid where it
# is large; `reduce_max` combines per-rank maxima (global dt of hydro)
def _heat3d_slab(sizes, lo, hi, reduce_max):
    from paper_1710_08774_b200 import inputs
    return [inputs.heat3d_planes(*sizes, lo, hi + 2)]


def _biharm_slab(sizes, lo, hi, reduce_max):
    return [np.ascontiguousarray(_biharm_inputs(sizes)[0][lo:hi + 4])]


def _box_slab(sizes, lo, hi, reduce_max):
    return [np.ascontiguousarray(_box_inputs(sizes)[0][lo:hi + 4])]


def _hydro_slab(sizes, lo, hi, reduce_max):
    from paper_1710_08774_b200 import inputs
    st, smax = inputs.hydro_rows(sizes[0], sizes[1], lo - 2, hi + 2)
    return st + [np.array([0.5 / reduce_max(smax)], dtype=np.float64)]


WORKLOADS = {
    "heat3d": dict(config_index=1, spec="heat3d", sizes=(512, 512, 512), chain_steps=50,
                   gen=_heat3d_inputs, slab=_heat3d_slab, dtype="f64", halo=(1, 1, True)),
    "biharm": dict(config_index=0, spec="biharmonic2d", sizes=(4096, 4096), chain_steps=100,
                   gen=_biharm_inputs, slab=_biharm_slab, dtype="f64", halo=(2, 2, False)),
    "box": dict(config_index=3, spec="box2x", sizes=(16384, 16384), chain_steps=1,
                gen=_box_inputs, slab=_box_slab, dtype="f32", halo=None),
    "hydro": dict(config_index=2, spec="hydro2d", sizes=(4096, 4096), chain_steps=20,
                  gen=_hydro_inputs, slab=_hydro_slab, dtype="f64", halo=(2, 2, False)),
    # BASELINE.json configs[4] -- the default bench line (the metric's 1/2/4/8-GPU grid)
    "hydro_large": dict(config_index=4, spec="hydro2d", sizes=(32768, 32768), chain_steps=10,
                        gen=_hydro_inputs, slab=_hydro_slab, dtype="f64", halo=(2, 2, False)),
    # configs[4] with the adaptive CFL time step (specs/hydro2d_adaptive.lf): one
    # MAX reduction per step fused into the executor (+ an all-reduce per step on N GPUs)
    "hydro_large_adaptive": dict(config_index=None, spec="hydro2d_adaptive", sizes=(32768, 32768), chain_steps=10,
                                 gen=_hydro_inputs, slab=_hydro_slab, dtype="f64", halo=(2, 2, False)),
    # configs[2] / configs[4] in place (config.aliases declared for every iterate pair,
    # goals passed on their axioms' buffers): one copy of the state instead of three
    "hydro_inplace": dict(config_index=2, spec="hydro2d", sizes=(4096, 4096), chain_steps=20, gen=_hydro_inputs,
                          slab=_hydro_slab, dtype="f64", halo=(2, 2, False), inplace=True, alias=True),
    "hydro_large_inplace": dict(config_index=4, spec="hydro2d", sizes=(32768, 32768), chain_steps=10,
                                gen=_hydro_inputs, slab=_hydro_slab, dtype="f64", halo=(2, 2, False), inplace=True,
                                alias=True),
    "biharm_inplace": dict(config_index=0, spec="biharmonic2d", sizes=(4096, 4096), chain_steps=100,
                           gen=_biharm_inputs, slab=None, dtype="f64", halo=(2, 2, False), inplace=True, alias=True),
    # the same chains written with `body:` expressions: the generic NVRTC path
    "heat3d_jit": dict(config_index=1, spec="examples/heat3d_body", sizes=(512, 512, 512), chain_steps=50,
                       gen=_heat3d_inputs, slab=_heat3d_slab, dtype="f64", halo=(1, 1, True)),
    "biharm_jit": dict(config_index=0, spec="examples/biharm_body", sizes=(4096, 4096), chain_steps=100,
                       gen=_biharm_inputs, slab=_biharm_slab, dtype="f64", halo=(2, 2, False)),
    "box_jit": dict(config_index=3, spec="examples/box_body", sizes=(16384, 16384), chain_steps=1,
                    gen=_box_inputs, slab=_box_slab, dtype="f32", halo=None),
    # multi-nest plan: row sums of squared differences (a reduction), their root,
    # and a broadcast divide -- 2 nests, 1 split (the paper's normalization example)
    "normalization_jit": dict(config_index=None, spec="examples/normalization_body", sizes=(8192, 8192),
                              chain_steps=1, gen=lambda sz, seed=0: _norm_inputs(sz, seed), slab=None,
                              dtype="f64", halo=None),
    # in place (config.aliases, one buffer for u and unew): half the footprint
    "heat3d_jit_inplace": dict(config_index=1, spec="examples/heat3d_inplace", sizes=(512, 512, 512),
                               chain_steps=50, gen=_heat3d_inputs, slab=None, dtype="f64", halo=(1, 1, True),
                               inplace=True),
    "biharm_jit_inplace": dict(config_index=0, spec="examples/biharm_inplace", sizes=(4096, 4096),
                               chain_steps=100, gen=_biharm_inputs, slab=None, dtype="f64", halo=(2, 2, False),
                               inplace=True),
}


def measured_peak():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


# Hydro2D: algorithmic flops per cell-step of the user kernels as written
# (oracle/flopcount.cpp, pinned by tests/test_flopcount.py; + - * / sqrt = 1)
HYDRO_FLOPS_PER_CELL_STEP = 853.3264


def measured_fp64_peak():
    """fp64 FMA-pipe TFLOP/s measured live by tools/libfp64probe.so (8 DFMA
    chains per thread, 8 CTAs of 256 per SM, best of 5)."""
    import ctypes
    lib = ctypes.CDLL(str(ROOT / "tools" / "libfp64probe.so"))
    out = ctypes.c_double(0.0)
    if lib.lf_probe_fp64_tflops(5, ctypes.byref(out)) != 0:
        raise RuntimeError("fp64 probe failed")
    return out.value


def ncu_pipe(workload):
    """fp64-pipe and issue-slot utilisation of the kernel from its newest committed ncu summary"""
    cands = sorted((ROOT / "profiles").glob(f"r0*_{workload}_ncu.json"))
    if not cands:
        return None
    p = cands[-1]
    d = json.loads(p.read_text())
    return {"fp64_pipe_pct": d.get("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"),
            "issue_active_pct": d.get("sm__issue_active.avg.pct_of_peak_sustained_elapsed"),
            "source": f"profiles/{p.name} (ncu --set full)"}


def ncu_traffic(workload):
    """DRAM bytes per launch from the committed ncu summary, if any."""
    p = ROOT / "profiles" / "traffic.json"
    if p.exists():
        d = json.loads(p.read_text())
        v = d.get(workload)
        if isinstance(v, dict):
            return v.get("dram_bytes_per_launch")
    return None


# --------------------------------------------------------------------- clocks
class ClockSampler:
    """Samples SM clock + throttle reasons through NVML during the timed region."""

    def __init__(self, index=0, period=0.02):
        self.samples, self.reasons = [], set()
        self.period, self.index = period, index
        self._stop = threading.Event()
        self.max_mhz = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        nv = self.nv
        names = {
            "hw_slowdown": getattr(nv, "nvmlClocksThrottleReasonHwSlowdown", 0x8),
            "hw_thermal_slowdown": getattr(nv, "nvmlClocksThrottleReasonHwThermalSlowdown", 0x40),
            "sw_thermal_slowdown": getattr(nv, "nvmlClocksThrottleReasonSwThermalSlowdown", 0x20),
            "sw_power_cap": getattr(nv, "nvmlClocksThrottleReasonSwPowerCap", 0x4),
            "hw_power_brake_slowdown": getattr(nv, "nvmlClocksThrottleReasonHwPowerBrakeSlowdown", 0x80),
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                for k, bit in names.items():
                    if r & bit:
                        self.reasons.add(k)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.nv is not None:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.nv is not None:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                    "samples": 0}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# --------------------------------------------------------------------- CPU legs
# bounded CPU samples of each workload: (rows of the outer dimension kept, ...)
# -- a full-width band for the 2D chains, a plane band for heat3d
NAIVE_SAMPLE = {"heat3d": (32, 512, 512), "biharm": (512, 4096), "box": (1024, 16384), "hydro": (16, None)}


def cpu_runner(name, w, naive=False):
    """One bounded unit of the workload on the CPU: the HFAV-style fused CPU
    schedule on all host threads (naive=False), or run_naive (R/SPEC.md:532-540,
    every intermediate materialised, one thread).  Both from oracle/ built with
    -march=native on this host.  Returns (run, cell-updates per run, threads, text)."""
    import oracle
    name = name.replace("_jit", "").replace("_inplace", "").replace("_large", "").replace("_adaptive", "")
    threads = 1 if naive else oracle.max_threads()
    sizes = w["sizes"]
    if naive:
        sizes = tuple(n if n is not None else sizes[-1] for n in NAIVE_SAMPLE.get(name, sizes))
    what = "run_naive" if naive else "fused CPU schedule"
    if name == "heat3d":
        u = w["gen"](sizes)[0]
        o = np.empty_like(u)
        run = (lambda: oracle.heat3d(u, 1, native=True)) if naive else \
            (lambda: oracle.heat3d_step(u, o, threads=threads, native=True))
        return run, int(np.prod(sizes)), threads, f"1 time step of {'x'.join(map(str, sizes))} ({what})"
    if name == "biharm":
        u = w["gen"](sizes)[0]
        o = np.zeros_like(u)
        run = (lambda: oracle.biharm(u, 1, native=True)) if naive else \
            (lambda: oracle.biharm_step(u, o, threads=threads, native=True))
        return run, int(np.prod(sizes)), threads, f"1 iteration of {'x'.join(map(str, sizes))} ({what})"
    if name == "box":
        img = w["gen"](sizes)[0]
        return (lambda: oracle.box(img, fused=not naive, threads=threads, native=True)), int(np.prod(sizes)), \
            threads, f"1 pass of {'x'.join(map(str, sizes))} ({what})"
    if name == "normalization":
        # numpy restatement of run_naive for this chain on a 512-row band (single thread)
        q, z = w["gen"]((512, sizes[1]))

        def run():
            fl = (q[:, 1:] - q[:, :-1]) * (q[:, 1:] - q[:, :-1])
            acc = z.copy()
            for i in range(fl.shape[1]):
                acc = acc + fl[:, i]
            return fl / np.sqrt(acc)[:, None]
        return run, 512 * sizes[1], 1, f"a 512x{sizes[1]} row band (numpy run_naive)"
    # hydro: a full-width row band, 1 step (x-sweep then y-sweep)
    nj = sizes[0] if naive else max(16, min(sizes[0], 64))
    st = w["gen"]((nj, sizes[1]))
    outs = [np.empty_like(a) for a in st[:4]]
    dtdx = float(st[4][0])
    run = (lambda: oracle.hydro(st[:4], dtdx, 1, native=True)) if naive else \
        (lambda: oracle.hydro_step(st[:4], outs, dtdx, threads=threads, native=True))
    return run, nj * sizes[1], threads, f"1 step of a {nj}x{sizes[1]} row band ({what})"


def cpu_sample(name, w, budget_s=10.0, naive=False):
    """Repeat the CPU unit for ~budget_s; returns (cell-updates/s, threads, text)."""
    run, cells, threads, unit = cpu_runner(name, w, naive=naive)
    run()  # warm
    t0 = time.perf_counter()
    reps = 0
    while True:
        run()
        reps += 1
        if time.perf_counter() - t0 >= budget_s:
            break
    dt = time.perf_counter() - t0
    return cells * reps / dt, threads, f"{reps} x {unit}, {threads} thread(s), {dt:.1f} s"


def host_cpu():
    """CPU model, physical cores, logical CPUs usable, OMP_NUM_THREADS."""
    try:
        import psutil
        phys = psutil.cpu_count(logical=False)
    except Exception:
        phys = None
    return {"cpu": cpu_model(), "physical_cores": phys, "logical_cpus": len(os.sched_getaffinity(0)),
            "omp_num_threads": os.environ.get("OMP_NUM_THREADS"),
            "build": "gcc -O3 -march=native -ffp-contract=off -fopenmp (oracle/, built on this host)"}


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"



# small grid and step count of the N-GPU self-check (dim 0 divisible by 1, 2, 4, 8)
PARITY_2D, PARITY_3D = ((512, 512), 3), ((64, 64, 64), 3)


def slab_parity(w, lf, comm, rank, world, dev, stream):
    """GPU(N) == GPU(1) on a small grid: every rank runs its slab through
    lf_run_slabs (the same NCCL exchange as the timed run), the interior rows
    are gathered to rank 0 and compared bit for bit with a whole-domain lf_run
    of the same input (ghost columns included).  Returns True/False on rank 0,
    None where the chain has no exchange."""
    import torch
    import torch.distributed as dist
    from paper_1710_08774_b200 import slabs
    if w["halo"] is None:
        return None
    sizes, steps = PARITY_3D if len(w["sizes"]) == 3 else PARITY_2D
    plan = lf.Plan.with_ranges(w["spec"], sizes, inplace=bool(w.get("alias")))
    n0 = sizes[0]
    lo, hi = slabs.slab_range(n0, rank, world)

    def reduce_max(x):
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())
    local = w["slab"](sizes, lo, hi, reduce_max)
    d_ax = [torch.from_numpy(np.ascontiguousarray(h)).to(dev) for h in local]
    d_goal = []
    for k, t in enumerate(plan.goals):
        if w.get("inplace"):  # the timed run's mode: goals on the axioms' slab buffers
            d_goal.append(d_ax[k])
            continue
        ext = list(t.extent)
        ext[0] = ext[0] - n0 + (hi - lo)
        d_goal.append(torch.full(ext, float("nan"), dtype=getattr(torch, str(t.dtype)), device=dev))
    plan.run_slabs(d_ax + d_goal, comm, steps=steps, stream=stream)
    torch.cuda.synchronize()
    g0 = [-t.base[0] for t in plan.goals]  # ghost rows before the slab's first row
    mine = torch.stack([g[o:o + (hi - lo)] for g, o in zip(d_goal, g0)])
    parts = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(parts, mine)
    if rank != 0:
        return None
    whole_in = w["gen"](sizes)
    ax = [torch.from_numpy(np.ascontiguousarray(h)).to(dev) for h in whole_in[:len(plan.axioms)]]
    goals = [torch.full(t.extent, float("nan"), dtype=getattr(torch, str(t.dtype)), device=dev) for t in plan.goals]
    plan.run(ax + goals, steps=steps, stream=stream)
    torch.cuda.synchronize()
    ref = torch.stack([g[o:o + n0] for g, o in zip(goals, g0)])
    got = torch.cat(parts, dim=1)
    return bool(torch.equal(got.view(torch.int64) if got.dtype == torch.float64 else got.view(torch.int32),
                            ref.view(torch.int64) if ref.dtype == torch.float64 else ref.view(torch.int32)))

# --------------------------------------------------------------------- main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="loomfuse", choices=["loomfuse", "reference"])
    ap.add_argument("--config", default="hydro_large", choices=sorted(WORKLOADS),
                    help="default: BASELINE configs[4], the grid the metric is quoted on (1/2/4/8 GPUs)")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-e2e", action="store_true", help="skip the end-to-end leg")
    ap.add_argument("--cpu-budget", type=float, default=10.0)
    ap.add_argument("--slab-exchange", choices=["native", "torch"], default="native",
                    help="multi-GPU halo exchange: lf_run_slabs (NCCL issued by the library, default) or "
                         "torch.distributed P2P around lf_run_slab")
    ap.add_argument("--force-slabs", action="store_true",
                    help="testing: run the multi-GPU slab path (overlapped NCCL schedule) even on one GPU")
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    w = WORKLOADS[args.config]
    cells = int(np.prod(w["sizes"]))
    metric = "fused-chain cell-updates/s"
    origin = f"BASELINE configs[{w['config_index']}]" if w["config_index"] is not None else "extra (not a BASELINE config)"
    workload = f"{origin} {w['spec']} " + "x".join(map(str, w["sizes"])) + \
        f", {w['chain_steps']} steps"
    slab_mode = world > 1 or args.force_slabs
    # one config dict for both arms (--impl loomfuse / reference): same keys, same values
    config = {"workload": workload, "l2": "inputs larger than L2 (126 MB)", "in_place": bool(w.get("inplace")),
              "parallelism": f"slab{world}" if slab_mode else "single-gpu"}

    if args.impl == "reference":
        if rank != 0:
            return
        run, unit_cells, threads, unit = cpu_runner(args.config, w)
        for _ in range(args.warmup):
            run()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            run()
        dt = (time.perf_counter() - t0) / args.steps
        value = unit_cells / dt
        sample = f"{args.steps} x {unit}, {threads} threads"
        line = {
            "impl": "reference", "metric": metric, "value": value, "unit": "cell-updates/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": dt * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": w["dtype"], "data": "synthetic (seeded splitmix64, BASELINE.json shapes)",
            "config": config, "executor": "HFAV fused CPU schedule (oracle/ port; the reference's executor is "
                                          "absent from the snapshot)",
            "cpu_baseline": {"value": value, "unit": "cell-updates/s", "cores": threads, "kind": "port",
                             "sample": sample, **host_cpu()},
            "e2e": {"value": value, "unit": "cell-updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        }
        print(json.dumps(line), flush=True)
        return

    import torch
    import paper_1710_08774_b200 as lf
    from paper_1710_08774_b200 import slabs

    # stdout carries exactly one JSON line: everything native code prints while
    # we run (the NCCL version banner of the first communicator, ...) goes to
    # stderr; the saved descriptor is restored for the final print
    sys.stdout.flush()
    json_fd = os.dup(1)
    os.dup2(2, 1)
    if slab_mode:
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        if world == 1:  # --force-slabs on one GPU: a one-rank NCCL group
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", str(29000 + os.getpid() % 1000))
            dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", local_rank))
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    else:
        torch.cuda.set_device(0)
    dev = torch.device("cuda", torch.cuda.current_device())

    plan = lf.Plan.with_ranges(w["spec"], w["sizes"], inplace=bool(w.get("alias")))
    if not plan.executor:
        raise SystemExit(f"no fused executor for {w['spec']}: run lf_run to see why")
    nax = len(plan.axioms)
    stream = torch.cuda.current_stream()
    tdt = lambda t: getattr(torch, str(t.dtype))

    # ---------------- device-resident timing ----------------
    if not slab_mode:
        host = w["gen"](w["sizes"])
        d_ax = [torch.from_numpy(h).to(dev) for h in host[:nax]]
        if w.get("inplace"):  # goal k shares axiom k's buffer
            d_goal = [d_ax[k] for k in range(len(plan.goals))]
        else:
            d_goal = [torch.empty(t.extent, dtype=tdt(t), device=dev) for t in plan.goals]
        bufs = d_ax + d_goal

        def one_step():
            plan.run(bufs, steps=w["chain_steps"], stream=stream)
    else:
        if w.get("inplace") and not (w.get("alias") and args.slab_exchange == "native"):
            raise SystemExit("in-place slab runs: the built-in Hydro2D executor through lf_run_slabs only")
        # outer-dimension slabs, faces exchanged by NCCL every time step
        n0 = w["sizes"][0]
        lo, hi = slabs.slab_range(n0, rank, world)

        def reduce_max(x):
            t = torch.tensor([x], dtype=torch.float64, device=dev)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            return float(t.item())
        host = None
        local = w["slab"](w["sizes"], lo, hi, reduce_max)
        d_ax = [torch.from_numpy(np.ascontiguousarray(h)).to(dev) for h in local]
        state = [i for i, t in enumerate(plan.axioms) if len(t.extent) > 0]
        d_goal = []
        for k, t in enumerate(plan.goals):
            if w.get("inplace"):  # every state goal on its axiom's slab buffer
                d_goal.append(d_ax[k])
                continue
            ext = list(t.extent)
            ext[0] = ext[0] - n0 + (hi - lo)  # same halo, local rows
            d_goal.append(torch.empty(ext, dtype=tdt(t), device=dev))
        if w["halo"] is None:  # no iterate pairs: independent slabs, halo rows replicated in the input
            def one_step():
                for _ in range(w["chain_steps"]):
                    plan.run_slab(d_ax + d_goal, lo, hi, n0, stream=stream)
        elif args.slab_exchange == "native":
            # lf_run_slabs: faces first, NCCL send/recv of the faces on the
            # library's side stream overlapped with the interior, per step
            comm = lf.NcclComm.from_group(rank, world)

            def one_step():
                plan.run_slabs(d_ax + d_goal, comm, steps=w["chain_steps"], stream=stream)
        else:
            halo = slabs.Halo(*w["halo"])
            cur = [d_ax[i] for i in state]
            nxt = [torch.empty_like(d_ax[i]) for i in state]

            def launch(src, dst, part):
                bufs = list(d_ax)
                for k, i in enumerate(state):
                    bufs[i] = src[k]
                plan.run_slab(bufs + list(dst), lo, hi, n0, stream=torch.cuda.current_stream(), part=part)

            comm = torch.cuda.Stream(device=dev, priority=-1)

            def one_step():
                # face rows first, their NCCL exchange overlapped with the interior rows
                slabs.run_slabs_overlapped(launch, cur, nxt, w["chain_steps"], halo, rank, world, hi - lo,
                                           comm_stream=comm)
    parity = None
    if slab_mode and w["halo"] is not None:
        # N-GPU self-check before timing (printed as "slab_parity")
        pcomm = comm if args.slab_exchange == "native" else lf.NcclComm.from_group(rank, world)
        parity = slab_parity(w, lf, pcomm, rank, world, dev, stream)
    # one pass over the grid per step, except where the executor fuses time
    # steps (heat3d: two-step passes on a whole domain); slabs step singly
    passes = plan.grid_passes(w["chain_steps"]) if not slab_mode else w["chain_steps"]
    if not slab_mode:
        launches = plan.launches(w["chain_steps"])
        if w.get("inplace"):  # + the band commit (or capture) kernel of every in-place step
            launches += w["chain_steps"]
    elif w["halo"] is None:
        launches = plan.launches_per_step * w["chain_steps"]
    else:
        # lf_run_slabs' schedule (capi.cpp run_slabs_core): `whole` -- one launch
        # per step -- for slabs of >= 1024 rows, else `parallel` -- the two face
        # parts and the interior, every step (LF_SLAB_SCHEDULE overrides)
        sched = os.environ.get("LF_SLAB_SCHEDULE") or ("whole" if hi - lo >= 1024 else "parallel")
        # the Python exchange path (slabs.run_slabs_overlapped) always splits faces / interior
        per_step = 1 if args.slab_exchange == "native" and sched == "whole" else 3
        if w.get("inplace"):
            per_step = 2  # whole-slab launches only: the step and its band commit
        launches = per_step * plan.launches_per_step * w["chain_steps"]

    def barrier():
        if slab_mode:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        one_step()
    barrier()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(torch.cuda.current_device()) as clk:
        barrier()
        start.record(stream)
        for _ in range(args.steps):
            one_step()
        end.record(stream)
        barrier()
    ms = start.elapsed_time(end) / args.steps
    if world > 1:
        t = torch.tensor([ms], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    value = cells * w["chain_steps"] / (ms / 1e3)

    # roofline of the dominant (only) kernel: algorithmic bytes per pass over
    # the grid (terminals read once + written once) / average pass duration
    # over the timed region (= per-launch bytes / launch time for one kernel
    # per pass)
    peak, peak_src = measured_peak()
    bpc = plan.compulsory_bytes_per_cell
    cells_local = cells / (world if world > 1 else 1)
    pass_s = (ms / 1e3) / max(1, passes)
    achieved = bpc * cells_local / pass_s / 1e9
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": ncu_traffic(args.config), "peak_source": peak_src,
                "algorithmic_bytes_per_cell": bpc, "cell_updates_per_pass": w["chain_steps"] / max(1, passes),
                "passes": passes}
    if w["spec"].startswith("hydro2d"):
        # compute-bound chain: the fp64 roofline is the binding one; HBM kept beside it
        fpk = measured_fp64_peak()
        tf = HYDRO_FLOPS_PER_CELL_STEP * cells_local * w["chain_steps"] / (ms / 1e3) / 1e12
        roofline = {"bound": "fp64", "achieved": tf, "peak": fpk, "unit": "TFLOP/s", "frac": tf / fpk,
                    "traffic": ncu_traffic(args.config),
                    "peak_source": "measured live (tools/fp64_probe.cu: DFMA chains)",
                    "algorithmic_flops_per_cell_step": HYDRO_FLOPS_PER_CELL_STEP,
                    "hbm": {"achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                            "algorithmic_bytes_per_cell": bpc, "peak_source": peak_src},
                    # each division / square root is ~10 fp64-pipe instructions: the
                    # pipe itself is far busier than the algorithmic-flop fraction
                    "pipe": ncu_pipe(args.config)}

    line = {
        "metric": metric, "value": value, "unit": "cell-updates/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": w["dtype"], "data": "synthetic (seeded splitmix64, BASELINE.json shapes)",
        "config": config, "executor": plan.executor,
        **({"halo_exchange": args.slab_exchange if w["halo"] is not None else "none"} if slab_mode else {}),
        "roofline": roofline, "gpu_launches": launches * args.steps, "clocks": clk.summary(),
    }
    if slab_mode:
        line["slab_parity"] = parity

    # ---------------- end-to-end through the host-buffer ABI call ----------------
    e2e_bytes = sum(t.bytes for t in plan.terminals)
    if not args.no_e2e and not slab_mode and e2e_bytes > 100e9:
        line["e2e"] = None
        line["e2e_skipped"] = f"{e2e_bytes / 1e9:.0f} GB of terminals: pinned host copies would not fit beside the device run"
    elif not args.no_e2e and not slab_mode:
        del d_ax, d_goal, bufs  # lf_run_host owns its own device buffers
        torch.cuda.empty_cache()
        pinned = [torch.from_numpy(h).pin_memory() for h in host[:nax]]
        if w.get("inplace"):
            outs = [pinned[k] for k in range(len(plan.goals))]
        else:
            outs = [torch.empty(t.extent, dtype=tdt(t)).pin_memory() for t in plan.goals]
        hb = [p.numpy() for p in pinned] + [o.numpy() for o in outs]
        # a step moves every terminal over PCIe: bound the repetitions on the big grids
        e2e_steps, e2e_warm = (min(args.steps, 3), 1) if e2e_bytes > 10e9 else (args.steps, max(1, args.warmup))
        for _ in range(e2e_warm):
            plan.run_host(hb, steps=w["chain_steps"])
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            plan.run_host(hb, steps=w["chain_steps"])
        e2e_s = (time.perf_counter() - t0) / e2e_steps
        line["e2e"] = {"value": cells * w["chain_steps"] / e2e_s, "unit": "cell-updates/s",
                       "h2d_bytes_per_step": int(sum(t.bytes for t in plan.axioms)),
                       "d2h_bytes_per_step": int(sum(t.bytes for t in plan.goals)),
                       "ms_per_step": e2e_s * 1e3, "steps": e2e_steps, "warmup": e2e_warm,
                       "api": "lf_run_host (pinned host buffers; H2D, every chain step, D2H inside the timed call)"}
    elif not args.no_e2e and slab_mode and w["halo"] is not None and args.slab_exchange == "native":
        # N GPUs end to end: every rank copies its slab's axioms up from pinned
        # host memory, runs lf_run_slabs, copies its goals back; max over ranks
        h_ax = [t.cpu().pin_memory() for t in d_ax]
        h_goal = [torch.empty(t.shape, dtype=t.dtype).pin_memory() for t in d_goal]

        def e2e_step():
            for hsrc, dst in zip(h_ax, d_ax):
                dst.copy_(hsrc, non_blocking=True)
            plan.run_slabs(d_ax + d_goal, comm, steps=w["chain_steps"], stream=stream)
            for src, hdst in zip(d_goal, h_goal):
                hdst.copy_(src, non_blocking=True)
            torch.cuda.synchronize()
        e2e_steps = min(args.steps, 3)
        e2e_step()
        barrier()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            e2e_step()
        barrier()
        e2e_s = torch.tensor([(time.perf_counter() - t0) / e2e_steps], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(e2e_s, op=torch.distributed.ReduceOp.MAX)
        e2e_s = float(e2e_s.item())
        h2d = torch.tensor([sum(t.numel() * t.element_size() for t in h_ax)], dtype=torch.float64, device=dev)
        d2h = torch.tensor([sum(t.numel() * t.element_size() for t in h_goal)], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(h2d)
        torch.distributed.all_reduce(d2h)
        line["e2e"] = {"value": cells * w["chain_steps"] / e2e_s, "unit": "cell-updates/s",
                       "h2d_bytes_per_step": int(h2d.item()), "d2h_bytes_per_step": int(d2h.item()),
                       "ms_per_step": e2e_s * 1e3, "steps": e2e_steps, "warmup": 1,
                       "api": "per rank: pinned H2D of the slab, lf_run_slabs (NCCL halo exchange), D2H; "
                              "max over ranks"}
    # ---------------- CPU baseline (rank 0, N=1 only) ----------------
    if rank == 0 and world == 1 and not args.no_cpu:
        rate, threads, sample = cpu_sample(args.config, w, budget_s=args.cpu_budget)
        line["cpu_baseline"] = {"value": rate, "unit": "cell-updates/s", "cores": threads, "kind": "port",
                                "sample": sample, **host_cpu()}
        if args.config != "normalization_jit":
            nrate, nthreads, nsample = cpu_sample(args.config, w, budget_s=args.cpu_budget / 2, naive=True)
            line["cpu_baseline"]["run_naive"] = {"value": nrate, "unit": "cell-updates/s", "cores": nthreads,
                                                 "sample": nsample}
    sys.stdout.flush()
    os.dup2(json_fd, 1)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if slab_mode:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
