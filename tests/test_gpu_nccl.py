"""The NCCL path of shard.combine on the B200 (one rank: the box has one GPU;
the N > 1 logic is covered by the gloo tests): the packed float64 [R, 4]
all-reduce runs through NCCL with the device_id binding bench.py uses, and
leaves a single rank's partials unchanged -- COUNT exactly."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

_SCRIPT = r"""
import os, socket, sys
sys.path.insert(0, {root!r})
import numpy as np, torch, torch.distributed as dist
s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK="0", WORLD_SIZE="1", LOCAL_RANK="0")
torch.cuda.set_device(0)
dist.init_process_group("nccl", init_method="env://", device_id=torch.device("cuda", 0))
from paper_2010_12548_b200 import workloads as W
from paper_2010_12548_b200.query import AggregationQuery, PreparedJoin
from paper_2010_12548_b200.shard import combine
w = W.c2(n=2_000_000)
prep = PreparedJoin(w.regions, AggregationQuery("SUM:fare", w.epsilon), w.grid)
r = prep.index.point_pass(torch.from_numpy(w.xy).cuda(), torch.from_numpy(w.attrs["fare"]).cuda()).check()
c0, s0 = r.cnt.clone(), r.sum.clone()
combine(r.cnt, r.sum, force=True)
torch.cuda.synchronize()
assert torch.equal(r.cnt, c0), "COUNT changed"
assert torch.allclose(r.sum, s0, rtol=0, atol=0), "SUM changed"
assert dist.get_backend() == "nccl"
dist.destroy_process_group()
print("ok")
"""


def test_combine_over_nccl():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    p = subprocess.run([sys.executable, "-c", _SCRIPT.format(root=ROOT)], capture_output=True, text=True, timeout=600)
    assert p.returncode == 0 and p.stdout.strip().endswith("ok"), p.stdout[-2000:] + p.stderr[-4000:]
