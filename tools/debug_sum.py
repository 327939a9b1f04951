import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle import oracle as O
from paper_2010_12548_b200 import workloads as W
from paper_2010_12548_b200.engine import ApproxIndex
from paper_2010_12548_b200.geometry import pack_regions
from paper_2010_12548_b200.grid import level_for_bound
n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 4_000_000
w = W.c2(n=n)
g = w.grid.with_level(level_for_bound(w.grid, w.epsilon))
p = pack_regions(w.regions)
A = O.Approx((g.origin.x, g.origin.y, g.extent, g.max_level), p.vx, p.vy, p.ring_off, p.poly_ring_off, p.poly_region, p.n_regions, 0)
co, so = A.join(w.xy, w.attrs['fare'], nthreads=16)
for layout in ('trie', 'dense'):
    idx = ApproxIndex(p, g, 0, layout=layout)
    r = idx.point_pass(w.xy, w.attrs['fare']).check()
    c = r.cnt.cpu().numpy(); s = r.sum.cpu().numpy()
    rel = np.abs(s - so) / np.maximum(np.abs(so), 1e-30)
    print(layout, 'count_eq', np.array_equal(c, co), 'max rel', rel.max(), 'alpha rel', rel[:, 0].max(), 'beta rel', rel[:, 1].max(),
          'tot', s.sum(), so.sum(), flush=True)
