"""Config-1 sample sharding through the PRODUCT on the GPU: two ranks as two processes
(gloo for the bookkeeping collectives) each solve their shard of seeded config-1 pairs
(n = 256, fp32 with the fp64 re-solve, reference gs.mu semantics) with the sm_100a
passes; the gathered per-pair maxima and means must equal a single-process solve of the
full index range bit for bit (sharding is invisible, no collective on the data path)."""
import dataclasses
import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]
PER_RANK = 48


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _solve(a, b):
    sys.path.insert(0, str(ROOT))
    from bench import greens_cfg1
    from paper_2307_12119_b200 import inputs
    from paper_2307_12119_b200.api import GT_FP32, DeviceGreens
    cfg = inputs.CONFIGS["cfg1"]
    p = inputs.power_batch(cfg, a, b - a, np.float32)
    v = inputs.variation_batch(cfg, a, b - a).numpy().astype(np.float32)
    dg = DeviceGreens(greens_cfg1(), GT_FP32)
    _, mx, mean, st, _ = dg.mc_batch_host(p, v, dg.opts(leak_frac=0.3, mu_per_sample=0), want_maps=False)
    dg.close()
    return mx, mean, st


def _worker(rank, world, port, q):
    sys.path.insert(0, str(ROOT))
    import torch
    import torch.distributed as dist
    from paper_2307_12119_b200 import shard
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    a, b = shard.shard_range(rank, world, PER_RANK)
    mx, mean, st = _solve(a, b)
    allmx = shard.gather_scalars(mx)
    allmean = shard.gather_scalars(mean)
    allst = shard.gather_scalars(st.astype(np.float64))
    if rank == 0:
        q.put((allmx, allmean, allst))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_product_sharding_matches_single(b200lib):
    import queue
    import torch.multiprocessing as mp
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = None
    while got is None:
        try:
            got = q.get(timeout=10)
        except queue.Empty:
            assert all(p.is_alive() or p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    mx1, mean1, st1 = _solve(0, world * PER_RANK)
    print(f"2-rank product sharding: {world * PER_RANK} pairs, max rise {mx1.min():.1f}..{mx1.max():.1f} K")
    assert (st1 == 0).all() and (got[2] == 0).all()
    np.testing.assert_array_equal(got[0], mx1)
    np.testing.assert_array_equal(got[1], mean1)
