"""Host-side enqueue cost of plan.run vs device time (is a config launch-bound?)."""
import sys, time
sys.path.insert(0, ".")
import torch
import paper_1710_08774_b200 as lf
from paper_1710_08774_b200 import inputs

for name, sizes, steps, gen in [("biharmonic2d", (4096, 4096), 100, lambda: [inputs.biharm_input(4096, 4096)]),
                                ("heat3d", (512, 512, 512), 50, lambda: [inputs.heat3d_input(512, 512, 512)])]:
    plan = lf.Plan.with_ranges(name, sizes)
    ax = [torch.from_numpy(a).cuda() for a in gen()]
    goals = [torch.empty(t.extent, dtype=torch.float64, device="cuda") for t in plan.goals]
    s = torch.cuda.current_stream()
    for _ in range(3):
        plan.run(ax + goals, steps=steps, stream=s)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    t0 = time.perf_counter()
    plan.run(ax + goals, steps=steps, stream=s)
    t1 = time.perf_counter()
    e1.record(s)
    torch.cuda.synchronize()
    print(name, "host enqueue us/launch", (t1 - t0) / steps * 1e6, "device us/launch", e0.elapsed_time(e1) / steps * 1e3)
