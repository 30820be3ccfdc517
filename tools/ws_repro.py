import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import paper_1710_08774_b200 as lf, oracle
from paper_1710_08774_b200 import inputs
shape = tuple(int(x) for x in sys.argv[1].split(','))
steps = int(sys.argv[2])
plan = lf.Plan.with_ranges("heat3d", shape)
u = inputs.heat3d_input(*shape, seed=4, sigma=3.0)
du = torch.from_numpy(u).cuda(); out = torch.full_like(du, float('nan'))
plan.run([du, out], steps=steps); torch.cuda.synchronize()
got = out.cpu().numpy()[1:-1,1:-1,1:-1]; ref = oracle.heat3d(u, steps)[1:-1,1:-1,1:-1]
print(shape, steps, plan.executor, 'OK' if np.array_equal(got.view(np.uint64), ref.view(np.uint64)) else 'MISMATCH %d' % np.count_nonzero(got != ref))
