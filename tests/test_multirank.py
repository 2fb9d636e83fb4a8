"""World-size-2 gloo run of the sharded Monte-Carlo bookkeeping (CPU only).

Each rank builds its shard of seeded config-1-generator pairs (n = 32), solves
it with the CPU oracle (the reference run_one), and the gathered per-pair
maxima must equal a single-process solve of the full index range: sharding is
invisible. max_over_ranks must return the slowest rank's time.
"""
import dataclasses
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, per_rank, out):
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import refpy
    from paper_2307_12119_b200 import inputs, shard
    d = refpy.calibrate(32, die_edge=0.016, beta=0.017, leak_total=84.0, fit_rand_scale=False)
    from paper_2307_12119_b200.api import GreensArrays
    g = GreensArrays(**{k: d[k] for k in ("n", "pitch", "f_sp0", "g_sp0", "phi", "kappa_inf", "alpha", "beta", "mu")})
    cfg = dataclasses.replace(inputs.CONFIGS["cfg1"], n=32, blocks=12)
    a, b = shard.shard_range(rank, world, per_rank)
    p = inputs.power_batch(cfg, a, b - a, np.float64)
    v = inputs.variation_batch(cfg, a, b - a).numpy().astype(np.float64)
    _, mx, _, st, _ = refpy.mc_batch(g, p, v, jobs=1, want_maps=False)
    allmx = shard.gather_scalars(mx)
    tmax = shard.max_over_ranks(float(rank + 1))
    if rank == 0:
        out.put((allmx.tolist(), tmax))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_sharding_matches_single(oracle):
    world, per_rank = 2, 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, per_rank, q)) for r in range(world)]
    for p in procs:
        p.start()
    gathered, tmax = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert tmax == 2.0
    from paper_2307_12119_b200 import inputs
    from paper_2307_12119_b200.api import GreensArrays
    d = oracle.calibrate(32, die_edge=0.016, beta=0.017, leak_total=84.0, fit_rand_scale=False)
    g = GreensArrays(**{k: d[k] for k in ("n", "pitch", "f_sp0", "g_sp0", "phi", "kappa_inf", "alpha", "beta", "mu")})
    cfg = dataclasses.replace(inputs.CONFIGS["cfg1"], n=32, blocks=12)
    p = inputs.power_batch(cfg, 0, world * per_rank, np.float64)
    v = inputs.variation_batch(cfg, 0, world * per_rank).numpy().astype(np.float64)
    _, mx, _, _, _ = oracle.mc_batch(g, p, v, jobs=2, want_maps=False)
    np.testing.assert_array_equal(np.array(gathered), mx)


def test_shard_ranges():
    from paper_2307_12119_b200.shard import shard_range
    assert [shard_range(r, 4, 10) for r in range(4)] == [(0, 10), (10, 20), (20, 30), (30, 40)]
    rs = [shard_range(r, 3, 0, weak=False, total=10) for r in range(3)]
    assert rs == [(0, 4), (4, 7), (7, 10)]
