"""bench.py's per-rank slab generators (the driver's N>1 runs): every slab's
storage rows equal the matching rows of the single-domain input, ghosts
included, and hydro's global dt is the single-domain one."""
import numpy as np
import pytest

import bench
from paper_1710_08774_b200 import slabs


@pytest.mark.parametrize("name,sizes", [("heat3d", (12, 8, 10)), ("biharm", (13, 9)), ("box", (11, 7)),
                                        ("hydro", (14, 9))])
@pytest.mark.parametrize("world", [2, 3])
def test_slab_generators_cut_the_global_input(name, sizes, world):
    w = bench.WORKLOADS[name]
    whole = w["gen"](sizes)
    halo = 1 if name == "heat3d" else 2
    maxes = []
    for rank in range(world):
        lo, hi = slabs.slab_range(sizes[0], rank, world)
        local = w["slab"](sizes, lo, hi, lambda x: (maxes.append(x), x)[1])
        for a, g in zip(local, whole):
            if g.ndim == 0 or g.shape == (1,):
                continue
            assert a.shape[0] == hi - lo + 2 * halo
            assert np.array_equal(a, g[lo:hi + 2 * halo]), (name, rank)
    if name == "hydro":
        # each rank passed its own maximum; the bench all-reduces them to the global one
        dts = [0.5 / m for m in maxes]
        assert np.isclose(min(dts), whole[4][0], rtol=0, atol=0)
