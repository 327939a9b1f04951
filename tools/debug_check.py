import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2010_12548_b200 import workloads as W
from paper_2010_12548_b200.engine import ApproxIndex
from paper_2010_12548_b200.geometry import pack_regions
from paper_2010_12548_b200.grid import level_for_bound
w = W.c2(n=4_000_000)
g = w.grid.with_level(level_for_bound(w.grid, w.epsilon))
p = pack_regions(w.regions)
idx = ApproxIndex(p, g, 0, layout='trie')
# debug build reports mismatches into cnt_out[0], cnt_out[1] (before the reduction adds real counts)
r = idx.point_pass(w.xy, w.attrs['fare'])
torch.cuda.synchronize()
print('raw cnt[0]', r.cnt.cpu().numpy()[0])
