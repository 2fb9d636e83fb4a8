"""Config 4 on the device: the four-step large-grid passes (large.cu) driven by
paper_2307_12119_b200/slab.py at world size 1, against the mode-B oracle
(oracle/restate.cpp ref_fixed_point_batch, fp64) and the batched mode-B kernels
on the same map. n = 512 (m = 1024 = 32 x 32) keeps the CPU oracle in seconds."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def greens512(b200lib, tmp_path_factory):
    from paper_2307_12119_b200.api import GreensArrays
    d = tmp_path_factory.mktemp("g512")
    n = 512
    (d / "stack.txt").write_text(f"n {n}\ndie_edge 0.016\n")
    (d / "var.txt").write_text("dopant_spread 0\nbeta 0.017\n")
    L = b200lib
    g = C.c_void_p()
    assert L.gt_calibrate(str(d / "stack.txt").encode(), str(d / "var.txt").encode(), None, 90.0, C.byref(g),
                          None) == 0, L.gt_last_error()
    maps = {}
    for k in ("f_sp0", "g_sp0"):
        f = C.c_void_p()
        assert L.gt_greens_field(g, k.encode(), C.byref(f)) == 0
        maps[k] = np.ctypeslib.as_array(L.gt_field_data(f), shape=(n, n)).copy()
        L.gt_field_free(f)
    f_sp0 = maps["f_sp0"]
    ga = GreensArrays(n=n, pitch=0.016 / n, f_sp0=f_sp0, g_sp0=maps["g_sp0"],
                      phi=float(np.mean(np.concatenate([f_sp0[0], f_sp0[-1], f_sp0[1:-1, 0], f_sp0[1:-1, -1]]))),
                      kappa_inf=float(f_sp0[0, 0]), alpha=L.gt_greens_alpha(g), beta=0.017, mu=L.gt_greens_mu(g),
                      rand_scale=1.0)
    L.gt_greens_free(g)
    return ga


@pytest.mark.parametrize("law,kirchhoff,beta", [(0, 0, 0.017), (1, 0, 0.004), (0, 1, 0.017)])
def test_large_grid_matches_oracle(b200lib, oracle, greens512, law, kirchhoff, beta):
    import torch
    from paper_2307_12119_b200 import inputs, slab
    from paper_2307_12119_b200.api import DeviceGreens
    cfg = inputs.CONFIGS["cfg4"]
    import dataclasses
    cfg = dataclasses.replace(cfg, n=512, blocks=64, hotspots=8)
    p = inputs.power_batch(cfg, 0, 1, np.float64) * 0.3
    v = inputs.variation_batch(cfg, 0, 1).numpy().astype(np.float64)
    kw = dict(leak_frac=0.3, beta=beta, law=law, kirchhoff=kirchhoff, tol=1e-4, max_iters=60)
    t_ref, it_ref, st_ref, secs = oracle.fixed_point_batch(greens512, p, v, jobs=1, **kw)
    assert st_ref[0] == 0
    dg = DeviceGreens(greens512, 1)
    ops = slab.GpuLargeOps(dg)
    o = dg.fp_opts(**kw)
    res = slab.solve_slab(ops, 512, torch.from_numpy(p[0]).cuda(), torch.from_numpy(v[0]).cuda(), o)
    torch.cuda.synchronize()
    t = res.t.cpu().numpy()
    err = np.abs(t - t_ref[0]).max()
    print(f"large n=512 law={law} kirchhoff={kirchhoff}: iters {res.iterations} vs {it_ref[0]}, "
          f"max|dT| {err:.3e} K on peak {t_ref.max():.1f} K (oracle {secs:.1f} s)")
    assert res.status == 0
    assert res.iterations == it_ref[0]
    assert err <= 1e-8
    # same map through the batched mode-B kernels (tile passes)
    out, it, st, _, _ = dg.fp_batch_host(p, v, o)
    assert it[0] == res.iterations
    assert np.abs(out[0] - t).max() <= 1e-9


def test_large_grid_needs_fp64(b200lib, greens512):
    from paper_2307_12119_b200 import slab
    from paper_2307_12119_b200.api import DeviceGreens, GtError
    dg = DeviceGreens(greens512, 0)
    with pytest.raises(GtError) as e:
        slab.GpuLargeOps(dg)
    assert e.value.status == 2


@pytest.mark.parametrize("n", [2048, 4096])
def test_large_grid_kernel_spectrum_n2048(b200lib, tmp_path, n):
    """n = 2048 / 4096 take the large-grid preparation (fk built by the four-step passes from
    the modal f_sp0; m = 4096 = 64 x 64 and 8192 = 128 x 64 column splits): three iterations
    against a direct numpy restatement."""
    import sys
    from pathlib import Path
    import torch
    from paper_2307_12119_b200 import slab
    from paper_2307_12119_b200.api import DeviceGreens, GreensArrays
    sys.path.insert(0, str(Path(__file__).parent))
    from slab_numpy_ops import baseline_fk, fixed_point_numpy, fixed_point_torch
    (tmp_path / "stack.txt").write_text(f"n {n}\ndie_edge 0.016\n")
    f = np.empty((n, n))
    nn = C.c_int()
    assert b200lib.gt_modal_kernel(str(tmp_path / "stack.txt").encode(), C.byref(nn),
                                   f.ctypes.data_as(C.POINTER(C.c_double))) == 0, b200lib.gt_last_error()
    assert nn.value == n and f.argmax() == (n // 2) * n + n // 2
    phi = float(np.mean(np.concatenate([f[0], f[-1], f[1:-1, 0], f[1:-1, -1]])))
    ga = GreensArrays(n=n, pitch=0.016 / n, f_sp0=f, g_sp0=f, phi=phi, kappa_inf=float(f[0, 0]), alpha=0.0,
                      beta=0.017, mu=0.0, rand_scale=1.0)
    rng = np.random.default_rng(5)
    P = rng.uniform(0.0, 4.0 / n ** 2 * 64, (n, n))
    V = 1.0 + 0.1 * rng.standard_normal((n, n))
    dg = DeviceGreens(ga, 1)
    o = dg.fp_opts(leak_frac=0.3, beta=0.017, law=0, kirchhoff=0, tol=1e-30, max_iters=3)
    res = slab.solve_slab(slab.GpuLargeOps(dg), n, torch.from_numpy(P).cuda(), torch.from_numpy(V).cuda(), o)
    torch.cuda.synchronize()
    if n <= 2048:
        ref, _ = fixed_point_numpy(P, V, baseline_fk(f, phi), 0.3, 0.017, 0, 1e-30, 3)
    else:  # the same restatement with torch.fft on the device (numpy would take minutes)
        ref, _ = fixed_point_torch(torch.from_numpy(P).cuda(), torch.from_numpy(V).cuda(), torch.from_numpy(f).cuda(),
                                   phi, 0.3, 0.017, 0, 1e-30, 3)
        ref = ref.cpu().numpy()
    err = np.abs(res.t.cpu().numpy() - ref).max()
    print(f"large n={n}: 3 iterations, max|dT| {err:.3e} K on peak {ref.max():.2f} K")
    assert res.iterations == 3 and res.status == slab.GT_SAMPLE_NOCONVERGE == 32
    assert err <= 1e-9 * max(1.0, ref.max())


def _large_greens(b200lib, tmp_path, n):
    from paper_2307_12119_b200.api import GreensArrays
    (tmp_path / "stack.txt").write_text(f"n {n}\ndie_edge 0.016\n")
    f = np.empty((n, n))
    nn = C.c_int()
    assert b200lib.gt_modal_kernel(str(tmp_path / "stack.txt").encode(), C.byref(nn),
                                   f.ctypes.data_as(C.POINTER(C.c_double))) == 0, b200lib.gt_last_error()
    phi = float(np.mean(np.concatenate([f[0], f[-1], f[1:-1, 0], f[1:-1, -1]])))
    return f, phi, GreensArrays(n=n, pitch=0.016 / n, f_sp0=f, g_sp0=f, phi=phi, kappa_inf=float(f[0, 0]),
                                alpha=0.0, beta=0.017, mu=0.0, rand_scale=1.0)


def test_config4_n8192_converged_vs_fp64_restatement(b200lib, tmp_path):
    """Config 4 at the benched size (n = 8192, m = 16384): the generator's map rescaled to
    300 W as in bench.py, leakage loop to 1e-4 K through slab.solve_slab, against a test-side
    fp64 restatement of the same loop with torch.fft (tests/slab_numpy_ops.fixed_point_torch):
    same iteration count, <= 1e-8 K."""
    import dataclasses
    import sys
    from pathlib import Path
    import torch
    from paper_2307_12119_b200 import inputs, slab
    from paper_2307_12119_b200.api import DeviceGreens
    sys.path.insert(0, str(Path(__file__).parent))
    from slab_numpy_ops import fixed_point_torch
    n = 8192
    f, phi, ga = _large_greens(b200lib, tmp_path, n)
    c4 = dataclasses.replace(inputs.CONFIGS["cfg4"], n=n)
    P = inputs.power_map_torch(c4, 0, device="cuda")
    P *= 300.0 / float(P.sum())
    V = inputs.variation_batch(c4, 0, 1, device="cuda", dtype=torch.float64)[0]
    dg = DeviceGreens(ga, 1)
    o = dg.fp_opts(leak_frac=0.3, beta=0.017, law=0, kirchhoff=0, tol=1e-4, max_iters=200)
    res = slab.solve_slab(slab.GpuLargeOps(dg), n, P, V, o)
    torch.cuda.synchronize()
    assert res.status == 0
    t_dev, it_dev = res.t.cpu().numpy(), res.iterations
    dg.close()
    del res
    torch.cuda.empty_cache()
    ref, it_ref = fixed_point_torch(P, V, torch.from_numpy(f).cuda(), phi, 0.3, 0.017, 0, 1e-4, 200)
    err = float(np.abs(t_dev - ref.cpu().numpy()).max())
    print(f"config 4 n=8192: {it_dev} iterations vs {it_ref} (restatement), max|dT| {err:.3e} K on peak "
          f"{float(ref.max()):.1f} K")
    assert it_dev == it_ref
    assert err <= 1e-8


def test_large_grid_n1024_converged_vs_oracle(b200lib, oracle, tmp_path):
    """The large-grid passes (four-step, m = 2048 = 32 x 64) through slab.solve_slab at
    n = 1024, converged to 1e-4 K, against the CPU oracle (reference outer loop with the
    reference's own baseline_kernel_spectrum convolution): same iterations, <= 1e-8 K."""
    import dataclasses
    import torch
    from paper_2307_12119_b200 import inputs, slab
    from paper_2307_12119_b200.api import DeviceGreens
    n = 1024
    f, phi, ga = _large_greens(b200lib, tmp_path, n)
    cfg = dataclasses.replace(inputs.CONFIGS["cfg4"], n=n, blocks=128, hotspots=16)
    p = inputs.power_batch(cfg, 0, 1, np.float64)
    p *= 300.0 / p.sum()
    v = inputs.variation_batch(cfg, 0, 1).numpy().astype(np.float64)
    kw = dict(leak_frac=0.3, beta=0.017, law=0, kirchhoff=0, tol=1e-4, max_iters=200)
    t_ref, it_ref, st_ref, secs = oracle.fixed_point_batch(ga, p, v, jobs=1, **kw)
    assert st_ref[0] == 0
    dg = DeviceGreens(ga, 1)
    res = slab.solve_slab(slab.GpuLargeOps(dg), n, torch.from_numpy(p[0]).cuda(), torch.from_numpy(v[0]).cuda(),
                          dg.fp_opts(**kw))
    torch.cuda.synchronize()
    err = float(np.abs(res.t.cpu().numpy() - t_ref[0]).max())
    print(f"large n=1024: iters {res.iterations} vs {it_ref[0]}, max|dT| {err:.3e} K on peak {t_ref.max():.1f} K "
          f"(oracle {secs:.1f} s)")
    assert res.status == 0 and res.iterations == it_ref[0]
    assert err <= 1e-8


def test_large_grid_n1024_chebyshev_vs_oracle(b200lib, oracle, tmp_path):
    """opts.accel on the large-grid path (Chebyshev steps in the inverse row pass, omega from
    slab.py): fewer iterations than the reference loop, same stop rule, and the result
    (G(x_k) of the last iteration) within 1e-3 K of the oracle's Picard fixed point."""
    import dataclasses
    import torch
    from paper_2307_12119_b200 import inputs, slab
    from paper_2307_12119_b200.api import DeviceGreens
    n = 1024
    f, phi, ga = _large_greens(b200lib, tmp_path, n)
    cfg = dataclasses.replace(inputs.CONFIGS["cfg4"], n=n, blocks=128, hotspots=16)
    p = inputs.power_batch(cfg, 0, 1, np.float64)
    p *= 300.0 / p.sum()
    v = inputs.variation_batch(cfg, 0, 1).numpy().astype(np.float64)
    kw = dict(leak_frac=0.3, beta=0.017, law=0, kirchhoff=0, tol=1e-4, max_iters=200)
    t_ref, it_ref, st_ref, _ = oracle.fixed_point_batch(ga, p, v, jobs=1, **kw)
    dg = DeviceGreens(ga, 1)
    o = dg.fp_opts(**kw)
    o.accel = 3
    res = slab.solve_slab(slab.GpuLargeOps(dg), n, torch.from_numpy(p[0]).cuda(), torch.from_numpy(v[0]).cuda(), o)
    torch.cuda.synchronize()
    err = float(np.abs(res.t.cpu().numpy() - t_ref[0]).max())
    print(f"large n=1024 Chebyshev: iters {res.iterations} vs {it_ref[0]} (Picard), max|dT| {err:.3e} K "
          f"on peak {t_ref.max():.1f} K")
    assert st_ref[0] == 0 and res.status == 0
    assert res.iterations < it_ref[0]
    assert err <= 1e-3


def test_large_grid_n1024_lowmode_anderson_vs_oracle(b200lib, oracle, tmp_path):
    """opts.accel = -3 on the large-grid path (slab._LowMode: Anderson(3) on the 16 x 16 lowest
    cosine modes of the row buffer between the column and inverse row phases): fewer
    iterations than the Chebyshev steps and the reference loop, same stop rule, within
    1e-3 K of the oracle's Picard fixed point."""
    import dataclasses
    import torch
    from paper_2307_12119_b200 import inputs, slab
    from paper_2307_12119_b200.api import DeviceGreens
    n = 1024
    f, phi, ga = _large_greens(b200lib, tmp_path, n)
    cfg = dataclasses.replace(inputs.CONFIGS["cfg4"], n=n, blocks=128, hotspots=16)
    p = inputs.power_batch(cfg, 0, 1, np.float64)
    p *= 300.0 / p.sum()
    v = inputs.variation_batch(cfg, 0, 1).numpy().astype(np.float64)
    kw = dict(leak_frac=0.3, beta=0.017, law=0, kirchhoff=0, tol=1e-4, max_iters=200)
    t_ref, it_ref, st_ref, _ = oracle.fixed_point_batch(ga, p, v, jobs=1, **kw)
    dg = DeviceGreens(ga, 1)
    its = {}
    for accel in (3, -3):
        o = dg.fp_opts(**kw)
        o.accel = accel
        res = slab.solve_slab(slab.GpuLargeOps(dg), n, torch.from_numpy(p[0]).cuda(), torch.from_numpy(v[0]).cuda(), o)
        torch.cuda.synchronize()
        assert res.status == 0
        its[accel] = res.iterations
    err = float(np.abs(res.t.cpu().numpy() - t_ref[0]).max())
    print(f"large n=1024 low-mode Anderson: iters {its[-3]} vs {its[3]} (Chebyshev) / {it_ref[0]} (Picard), "
          f"max|dT| {err:.3e} K on peak {t_ref.max():.1f} K")
    assert st_ref[0] == 0
    assert its[-3] < its[3] < it_ref[0]
    assert err <= 1e-3


@pytest.mark.parametrize("world,accel", [(2, 0), (4, 0), (4, 3), (4, -3), (8, 0)])
def test_large_grid_peer_ranks_emulated(b200lib, tmp_path, world, accel):
    """The multi-GPU column phase over peer memory (gt_large_cols_peer: every rank's row
    spectra read in place, results stored into their owners' row buffers), with `world`
    ranks emulated in one process on one GPU (slab.solve_slab_emulated): identical to the
    single-slab solve -- same iterations, same bits."""
    import dataclasses
    import torch
    from paper_2307_12119_b200 import inputs, slab
    from paper_2307_12119_b200.api import DeviceGreens
    n = 1024
    f, phi, ga = _large_greens(b200lib, tmp_path, n)
    cfg = dataclasses.replace(inputs.CONFIGS["cfg4"], n=n, blocks=128, hotspots=16)
    p = inputs.power_batch(cfg, 0, 1, np.float64)
    p *= 300.0 / p.sum()
    v = inputs.variation_batch(cfg, 0, 1).numpy().astype(np.float64)
    dg = DeviceGreens(ga, 1)
    o = dg.fp_opts(leak_frac=0.3, beta=0.017, law=0, kirchhoff=0, tol=1e-4, max_iters=200)
    o.accel = accel
    ops = slab.GpuLargeOps(dg)
    P, V = torch.from_numpy(p[0]).cuda(), torch.from_numpy(v[0]).cuda()
    one = slab.solve_slab(ops, n, P, V, o)
    em = slab.solve_slab_emulated(ops, n, P, V, o, world)
    torch.cuda.synchronize()
    d = float((em.t - one.t).abs().max())
    print(f"peer ranks emulated world={world} accel={accel}: iters {em.iterations} vs {one.iterations}, "
          f"max|dT| {d:.3e} K")
    assert em.status == one.status == 0
    assert em.iterations == one.iterations
    # low-mode mixing sums the ranks' partial projections in another order than one slab does
    assert d == 0.0 if accel >= 0 else d <= 1e-9
