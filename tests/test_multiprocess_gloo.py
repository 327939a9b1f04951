"""Multi-rank combine path on CPU (gloo, world_size 2): every rank joins its
point shard (the oracle stands in for the per-GPU pass here), the product's
shard.combine all-reduces the [R,2] partials, and the result equals the
single-process join -- COUNT exactly."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as O
        from paper_2010_12548_b200 import workloads as W
        from paper_2010_12548_b200.geometry import pack_regions
        from paper_2010_12548_b200.grid import level_for_bound
        from paper_2010_12548_b200.shard import combine, shard_range

        w = W.c1(n=200_000)
        L = level_for_bound(w.grid, w.epsilon)
        p = pack_regions(w.regions)
        A = O.Approx((w.grid.origin.x, w.grid.origin.y, w.grid.extent, L), p.vx, p.vy, p.ring_off,
                     p.poly_ring_off, p.poly_region, p.n_regions, 0)
        attr = np.random.default_rng(0).random(w.n).astype(np.float32)
        a, b = shard_range(w.n, rank, world)
        cnt, sm = A.join(w.xy[a:b], attr[a:b])
        tc, ts = torch.from_numpy(cnt), torch.from_numpy(sm)
        combine(tc, ts)
        if rank == 0:
            full_c, full_s = A.join(w.xy, attr)
            out.put((bool(np.array_equal(tc.numpy(), full_c)),
                     float(np.max(np.abs(ts.numpy() - full_s) / np.maximum(np.abs(full_s), 1e-30)))))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_combine_equals_single_process():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(240)
    assert all(p.exitcode == 0 for p in procs)
    ok, rel = q.get(timeout=5)
    assert ok
    assert rel < 1e-12
