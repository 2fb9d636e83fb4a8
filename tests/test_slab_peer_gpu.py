"""Config-4 multi-rank transports across PROCESSES on one GPU: the peer transport (CUDA IPC
mapped buffers, gloo barriers), and the copy ("nccl") transport with its all-to-all carried
by gloo through host memory. With the peer transport each rank's row spectra and row buffer are
cudaMalloc'ed and opened by the other rank (gt_ipc_open); the column kernels read the
other rank's spectra and store into its row buffer directly. Phases are separated by a
device sync + barrier on the host, so no kernel waits on another (B200_PROFILING: no
spinning ranks on one GPU). The result must equal the single-process solve bit for bit."""
import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _setup(n):
    import ctypes as C
    import dataclasses
    import tempfile
    from paper_2307_12119_b200 import inputs
    from paper_2307_12119_b200.api import GreensArrays, lib
    d = Path(tempfile.mkdtemp())
    (d / "stack.txt").write_text(f"n {n}\ndie_edge 0.016\n")
    f = np.empty((n, n))
    nn = C.c_int()
    L = lib()
    assert L.gt_modal_kernel(str(d / "stack.txt").encode(), C.byref(nn), f.ctypes.data_as(C.POINTER(C.c_double))) == 0
    phi = float(np.mean(np.concatenate([f[0], f[-1], f[1:-1, 0], f[1:-1, -1]])))
    ga = GreensArrays(n=n, pitch=0.016 / n, f_sp0=f, g_sp0=f, phi=phi, kappa_inf=float(f[0, 0]), alpha=0.0,
                      beta=0.017, mu=0.0, rand_scale=1.0)
    cfg = dataclasses.replace(inputs.CONFIGS["cfg4"], n=n, blocks=64, hotspots=8)
    p = inputs.power_batch(cfg, 0, 1, np.float64)[0]
    p *= 150.0 / p.sum()
    v = inputs.variation_batch(cfg, 0, 1).numpy().astype(np.float64)[0]
    return ga, p, v


def _gloo_exchange(out, inp, out_splits, in_splits):
    """all_to_all_single for CUDA tensors over gloo (host round trip): the copy transport's
    exchange logic with the device kernels, two processes on one GPU."""
    import torch.distributed as dist
    o = out.cpu()
    dist.all_to_all_single(o, inp.cpu(), out_splits, in_splits)
    out.copy_(o)


def _worker(rank, world, port, n, accel, q, transport="peer"):
    sys.path.insert(0, str(ROOT))
    import torch
    import torch.distributed as dist
    from paper_2307_12119_b200 import slab
    from paper_2307_12119_b200.api import DeviceGreens
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    ga, p, v = _setup(n)
    rows = n // world
    dg = DeviceGreens(ga, 1)
    o = dg.fp_opts(leak_frac=0.3, beta=0.017, law=0, kirchhoff=0, tol=1e-4, max_iters=100)
    o.accel = accel
    sl = slice(rank * rows, (rank + 1) * rows)
    res = slab.solve_slab(slab.GpuLargeOps(dg), n, torch.from_numpy(p[sl].copy()).cuda(),
                          torch.from_numpy(v[sl].copy()).cuda(), o, rank=rank, world=world, transport=transport,
                          exchange=_gloo_exchange if transport == "nccl" else None)
    torch.cuda.synchronize()
    q.put((rank, res.t.cpu().numpy(), res.iterations, res.status))
    dist.destroy_process_group()


@pytest.mark.parametrize("accel,transport", [(0, "peer"), (3, "peer"), (-3, "peer"), (0, "nccl")])
def test_peer_transport_two_processes(b200lib, accel, transport):
    import queue
    import torch
    import torch.multiprocessing as mp
    from paper_2307_12119_b200 import slab
    from paper_2307_12119_b200.api import DeviceGreens
    n, world = 512, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, accel, q, transport)) for r in range(world)]
    for p in procs:
        p.start()
    got = []
    while len(got) < world:
        try:
            got.append(q.get(timeout=10))
        except queue.Empty:
            assert all(p.is_alive() or p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    got.sort(key=lambda g: g[0])
    T = np.concatenate([g[1] for g in got])
    ga, pm, vm = _setup(n)
    dg = DeviceGreens(ga, 1)
    o = dg.fp_opts(leak_frac=0.3, beta=0.017, law=0, kirchhoff=0, tol=1e-4, max_iters=100)
    o.accel = accel
    one = slab.solve_slab(slab.GpuLargeOps(dg), n, torch.from_numpy(pm).cuda(), torch.from_numpy(vm).cuda(), o)
    d = float(np.abs(T - one.t.cpu().numpy()).max())
    print(f"{transport} transport, 2 processes, accel={accel}: iters {[g[2] for g in got]} vs {one.iterations}, "
          f"max|dT| {d:.3e} K")
    assert all(g[3] == 0 for g in got) and one.status == 0
    assert all(g[2] == one.iterations for g in got)
    # the low-mode mixing (accel < 0) all-reduces the ranks' partial projections: same steps to rounding
    assert d == 0.0 if accel >= 0 else d <= 1e-9
