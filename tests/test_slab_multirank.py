"""Config-4 slab decomposition, exchange logic on CPU ranks (gloo, world 2):
paper_2307_12119_b200/slab.py with the numpy stand-in phases
(tests/slab_numpy_ops.py, same buffer layouts as the gt_large_* kernels)
against a direct 2-D numpy restatement of the fixed point."""
import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n, q, accel=0, dct=False):
    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ROOT / "tests"))
    import torch
    import torch.distributed as dist
    from slab_numpy_ops import NumpyLargeOps, baseline_fk
    from paper_2307_12119_b200 import slab
    from paper_2307_12119_b200.api import FPOpts
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    z = np.load(ROOT / "tests" / "golden" / "greens_n64.npz")
    fk = baseline_fk(z["f_sp0"], float(z["phi"]))
    rng = np.random.default_rng(3)
    P = rng.uniform(0.0, 0.05, (n, n))
    V = 1.0 + 0.1 * rng.standard_normal((n, n))
    rows = n // world
    sl = slice(rank * rows, (rank + 1) * rows)
    o = FPOpts()
    o.leak_frac, o.law, o.kirchhoff, o.beta, o.tol, o.max_iters = 0.3, 0, 0, 0.017, 1e-10, 60
    o.t_ambient, o.eta = 318.15, 1.3
    o.accel = accel
    res = slab.solve_slab(NumpyLargeOps(n, fk, dct_rows=dct), n, torch.from_numpy(P[sl].copy()), torch.from_numpy(V[sl].copy()), o,
                          rank=rank, world=world)
    q.put((rank, res.t.numpy(), res.iterations, res.status))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,dct", [(1, False), (2, False), (2, True)])
def test_slab_exchange_matches_full_solve(world, dct):
    import torch.multiprocessing as mp
    sys.path.insert(0, str(ROOT / "tests"))
    from slab_numpy_ops import baseline_fk, fixed_point_numpy
    n = 64
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, q, 0, dct)) for r in range(world)]
    for p in procs:
        p.start()
    import queue
    got = []
    while len(got) < world:
        try:
            got.append(q.get(timeout=5))
        except queue.Empty:
            assert all(p.is_alive() or p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    got.sort(key=lambda g: g[0])
    T = np.concatenate([g[1] for g in got])
    z = np.load(ROOT / "tests" / "golden" / "greens_n64.npz")
    fk = baseline_fk(z["f_sp0"], float(z["phi"]))
    rng = np.random.default_rng(3)
    P = rng.uniform(0.0, 0.05, (n, n))
    V = 1.0 + 0.1 * rng.standard_normal((n, n))
    ref, it = fixed_point_numpy(P, V, fk, 0.3, 0.017, 0, 1e-10, 60)
    assert all(g[3] == 0 for g in got)
    assert all(g[2] == it for g in got), (it, [g[2] for g in got])
    assert np.abs(T - ref).max() < 1e-9


def _run(world, n, accel, dct=False):
    import queue
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, q, accel, dct)) for r in range(world)]
    for p in procs:
        p.start()
    got = []
    while len(got) < world:
        try:
            got.append(q.get(timeout=5))
        except queue.Empty:
            assert all(p.is_alive() or p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    got.sort(key=lambda g: g[0])
    return np.concatenate([g[1] for g in got]), [g[2] for g in got], [g[3] for g in got]


def test_slab_chebyshev_across_ranks():
    """opts.accel: every rank takes the same Chebyshev steps (omega from the max-over-ranks
    residual), so world 2 reproduces world 1 exactly, in fewer iterations than Picard,
    and lands on the Picard fixed point."""
    sys.path.insert(0, str(ROOT / "tests"))
    from slab_numpy_ops import baseline_fk, fixed_point_numpy
    n = 64
    t1, it1, st1 = _run(1, n, 3)
    t2, it2, st2 = _run(2, n, 3, dct=True)
    z = np.load(ROOT / "tests" / "golden" / "greens_n64.npz")
    fk = baseline_fk(z["f_sp0"], float(z["phi"]))
    rng = np.random.default_rng(3)
    P = rng.uniform(0.0, 0.05, (n, n))
    V = 1.0 + 0.1 * rng.standard_normal((n, n))
    ref, it = fixed_point_numpy(P, V, fk, 0.3, 0.017, 0, 1e-10, 60)
    assert st1 == [0] and st2 == [0, 0]
    assert it2 == [it1[0]] * 2 and it1[0] < it, (it1, it2, it)
    assert np.abs(t2 - t1).max() <= 1e-12
    assert np.abs(t1 - ref).max() <= 1e-8


def test_slab_lowmode_anderson_across_ranks():
    """opts.accel = -m: Anderson(m) on the 16 x 16 lowest cosine modes of the row buffer
    (slab._LowMode; partial projections all-reduced over the ranks' row slabs). World 2 takes
    the same steps as world 1 (same iteration count, same field to rounding), needs fewer
    iterations than Picard and lands on the Picard fixed point."""
    sys.path.insert(0, str(ROOT / "tests"))
    from slab_numpy_ops import baseline_fk, fixed_point_numpy
    n = 64
    t1, it1, st1 = _run(1, n, -3)
    t2, it2, st2 = _run(2, n, -3, dct=True)
    z = np.load(ROOT / "tests" / "golden" / "greens_n64.npz")
    fk = baseline_fk(z["f_sp0"], float(z["phi"]))
    rng = np.random.default_rng(3)
    P = rng.uniform(0.0, 0.05, (n, n))
    V = 1.0 + 0.1 * rng.standard_normal((n, n))
    ref, it = fixed_point_numpy(P, V, fk, 0.3, 0.017, 0, 1e-10, 60)
    print(f"low-mode Anderson(3): {it1[0]} iterations (world 1), {it2} (world 2), Picard {it}")
    assert st1 == [0] and st2 == [0, 0]
    assert it2 == [it1[0]] * 2 and it1[0] < it, (it1, it2, it)
    assert np.abs(t2 - t1).max() <= 1e-9
    assert np.abs(t1 - ref).max() <= 1e-8
