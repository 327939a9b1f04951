"""The product's multi-rank step with two ranks (world_size 2) on the one GPU
this pool provides: each rank runs the CUDA point pass on its contiguous point
shard (shard.shard_range) and shard.combine all-reduces the packed [R,4] float64
partials (gloo over the ranks' CUDA tensors; NCCL on a multi-GPU box).  The
ranks never wait on each other inside a kernel.  The combined COUNT equals the
oracle's bit-exactly; SUM within rel 1e-6."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, layout, out):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2010_12548_b200 import workloads as W
        from paper_2010_12548_b200.query import AggregationQuery, PreparedJoin
        from paper_2010_12548_b200.shard import combine, shard_range

        w = W.voronoi_tiling(3000, 1.0, seed=4, verts=(10, 30))
        rng = np.random.default_rng(0)
        n = 2_000_001
        xy = rng.random((n, 2))
        fare = rng.lognormal(2.5, 0.6, n).astype(np.float32)
        from paper_2010_12548_b200.grid import GridConfig

        prep = PreparedJoin(w, AggregationQuery(("SUM", "fare"), epsilon=1.0 / 4096 * 1.4142135623730951),
                            GridConfig((0.0, 0.0), 1.0, 0), layout=layout)
        a, b = shard_range(n, rank, world)
        r = prep.index.point_pass(torch.from_numpy(xy[a:b]).cuda(), torch.from_numpy(fare[a:b]).cuda()).check()
        combine(r.cnt, r.sum)
        torch.cuda.synchronize()
        if rank == 0:
            out.put((r.cnt.cpu().numpy(), r.sum.cpu().numpy(), prep.grid.max_level))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(600)
@pytest.mark.parametrize("layout", ["trie", "packed"])
def test_two_ranks_on_one_gpu_equal_oracle(oracle_lib, layout):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp

    from helpers import oracle_approx
    from paper_2010_12548_b200 import workloads as W
    from paper_2010_12548_b200.grid import GridConfig

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, layout, q)) for r in range(2)]
    for p in procs:
        p.start()
    cnt, sm, L = q.get(timeout=500)
    for p in procs:
        p.join(120)
    assert all(p.exitcode == 0 for p in procs)
    regions = W.voronoi_tiling(3000, 1.0, seed=4, verts=(10, 30))
    rng = np.random.default_rng(0)
    xy = rng.random((2_000_001, 2))
    fare = rng.lognormal(2.5, 0.6, len(xy)).astype(np.float32)
    A, _ = oracle_approx(oracle_lib, regions, GridConfig((0.0, 0.0), 1.0, L), 0)
    cnt_o, sum_o = A.join(xy, fare, nthreads=8)
    np.testing.assert_array_equal(cnt, cnt_o)
    np.testing.assert_allclose(sm, sum_o, rtol=1e-6, atol=1e-9)
