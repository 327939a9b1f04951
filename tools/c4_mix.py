"""C4 point composition (diagnostic): how the auto-selected hot slots and the
owner kinds split the points.  usage: python tools/c4_mix.py [points]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2010_12548_b200 import _native as N
from paper_2010_12548_b200 import workloads as W
from paper_2010_12548_b200.query import AggregationQuery, PreparedJoin

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 20_000_000
w = W.c4(n=n)
prep = PreparedJoin(w.regions, AggregationQuery("SUM:fare", w.epsilon), w.grid)
xy = torch.from_numpy(w.xy).cuda()
idx = prep.index
idx.auto_hot(xy)
v = idx.lookup(xy[: min(n, 4_000_000)]).to(torch.int64) & 0xFFFFFFFF
tot = len(v)
lst = (v & N.VALUE_LIST) != 0
single = (v != 0) & ~lst
code = v & N.CODE_MASK
bnd = single & ((code - 1) & 1).bool()
ishot = torch.zeros(idx.n_regions + 1, dtype=torch.bool, device=v.device)
ishot[torch.as_tensor(idx._hot, dtype=torch.int64, device=v.device)] = True
reg = torch.where(single, (code - 1) >> 1, torch.full_like(code, idx.n_regions))
hot = single & ~bnd & ishot[reg]
cold = single & ~bnd & ~ishot[reg]
for name, m in (("none", v == 0), ("list", lst), ("boundary single", bnd), ("interior hot", hot), ("interior cold", cold)):
    print(f"{name:16s} {m.sum().item() / tot:.4f}")
print(prep.stats())
