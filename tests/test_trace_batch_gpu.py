"""Config 3 (batched transient traces with the leakage update every step):
the device recursion path (trace_batch.cu) against the oracle, which drives the
reference's own time_varying_profile (solver.cpp:212-287) one step at a time
with P_n = P_dyn,n + L0 f(T_{n-1}) (oracle/restate.cpp ref_trace_leak_batch).
"""
import dataclasses

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _traces(B, steps, n=64, blocks=16, switch_prob=0.2, shared_blk=False):
    from paper_2307_12119_b200 import inputs
    cfg = dataclasses.replace(inputs.CONFIGS["cfg3"], n=n, blocks=blocks)
    blks, scheds, ons = [], [], []
    for b in range(B):
        blk, sched, on = inputs.markov_blocks(cfg, 0 if shared_blk else b, steps, switch_prob=switch_prob)
        if shared_blk and b:
            # same floorplan, independent chains: reuse block 0's map, reshuffle the schedule
            rng = np.random.default_rng(b)
            sched = sched[:, rng.permutation(sched.shape[1])]
        blks.append(blk)
        scheds.append(sched)
        ons.append(on)
    nblk = max(s.shape[1] for s in scheds)
    sched = np.zeros((B, steps, nblk))
    for b, s in enumerate(scheds):
        sched[b, :, :s.shape[1]] = s
    blk = np.stack(blks[:1] if shared_blk else blks)
    on = np.stack(ons)
    return blk, sched, on


def _run_gpu(greens, prec, blk, sched, leak0, dt, window, law, beta, out_stride):
    import torch
    from paper_2307_12119_b200.api import DeviceGreens
    dt_t = torch.float64 if prec else torch.float32
    B, steps, nblk = sched.shape
    n = greens.n
    dg = DeviceGreens(greens, prec)
    blk_d = torch.from_numpy(np.ascontiguousarray(blk, np.int32)).cuda()
    sch_d = torch.from_numpy(sched).to(dt_t).cuda()
    l0_d = torch.from_numpy(leak0).to(dt_t).cuda()
    frames = steps // out_stride
    out = torch.zeros((B, frames, n, n), dtype=dt_t, device="cuda")
    mx = torch.zeros((B, frames), dtype=torch.float64, device="cuda")
    o = dg.trace_opts(dt=dt, steps=steps, window=window, law=law, beta=beta, out_stride=out_stride)
    dg.trace_batch_device(blk_d.data_ptr(), n * n if blk.shape[0] > 1 else 0, sch_d.data_ptr(), nblk,
                          l0_d.data_ptr(), n * n if leak0.shape[0] > 1 else 0, B, o, out.data_ptr(), mx.data_ptr())
    torch.cuda.synchronize()
    return out.double().cpu().numpy(), mx.cpu().numpy()


@pytest.mark.parametrize("window,law,beta,shared", [(6, 0, 0.017, False), (40, 0, 0.017, True), (6, 1, 0.004, True)])
def test_trace_batch_matches_oracle(b200lib, oracle, greens64, window, law, beta, shared):
    """window < steps exercises the saturated tail (the r^(k+1) term); window > steps clips to steps.
    The exp law runs away at beta = 0.017 on these maps (as in mode B), so it is checked at 0.004."""
    B, steps, dt, stride = 3, 24, 2e-4, 4
    blk, sched, on = _traces(B, steps, shared_blk=shared)
    rng = np.random.default_rng(7)
    leak0 = 0.3 * on * rng.uniform(0.9, 1.1, size=on.shape)
    ref, st, secs = oracle.trace_leak_batch(greens64, blk, sched, leak0, dt, window, law=law, beta=beta,
                                            out_stride=stride)
    assert (st == 0).all(), st
    for prec, atol in ((1, 1e-8), (0, 1e-3)):
        out, mx = _run_gpu(greens64, prec, blk, sched, leak0, dt, window, law, beta, stride)
        err = np.abs(out - ref).max()
        print(f"window={window} law={law} prec={prec}: max|dT| {err:.3e} K on peak {ref.max():.2f} K "
              f"(oracle {secs:.2f} s)")
        assert err <= atol
        np.testing.assert_allclose(mx, out.reshape(B, steps // stride, -1).max(axis=2), rtol=0, atol=1e-12)


def test_trace_batch_without_capacitance_is_solver_error(b200lib, greens64):
    import ctypes as C
    from paper_2307_12119_b200.api import DeviceGreens, GtError
    g0 = dataclasses.replace(greens64, capacitance=0.0)
    blk, sched, on = _traces(1, 4)
    with pytest.raises(GtError) as e:
        _run_gpu(g0, 1, blk, sched, 0.3 * on, 2e-4, 2, 0, 0.017, 2)
    assert e.value.status == 3


def test_trace_batch_chunking_window1_and_ragged_stride(b200lib, oracle, greens64):
    """window = 1 (tail term every step), steps not a multiple of out_stride (trailing steps
    unstored), traces split over several in-flight chunks: same frames as the oracle."""
    import torch
    from paper_2307_12119_b200.api import DeviceGreens
    B, steps, dt, stride = 5, 11, 2e-4, 3
    blk, sched, on = _traces(B, steps)
    leak0 = 0.3 * on
    ref, st, _ = oracle.trace_leak_batch(greens64, blk, sched, leak0, dt, 1, law=0, beta=0.017, out_stride=stride)
    assert (st == 0).all()
    dg = DeviceGreens(greens64, 1)
    n = greens64.n
    blk_d = torch.from_numpy(blk).cuda()
    sch_d = torch.from_numpy(sched).cuda()
    l0_d = torch.from_numpy(leak0).cuda()
    out = torch.zeros((B, steps // stride, n, n), dtype=torch.float64, device="cuda")
    o = dg.trace_opts(dt=dt, steps=steps, window=1, law=0, beta=0.017, out_stride=stride, chunk=2)
    dg.trace_batch_device(blk_d.data_ptr(), n * n, sch_d.data_ptr(), sched.shape[2], l0_d.data_ptr(), n * n, B, o,
                          out.data_ptr())
    torch.cuda.synchronize()
    assert np.abs(out.cpu().numpy() - ref).max() <= 1e-8


def test_trace_batch_rejects_bad_options(b200lib, greens64):
    import torch
    from paper_2307_12119_b200.api import DeviceGreens, GtError
    dg = DeviceGreens(greens64, 1)
    blk, sched, on = _traces(1, 4)
    n = greens64.n
    blk_d = torch.from_numpy(blk).cuda()
    sch_d = torch.from_numpy(sched).cuda()
    l0_d = torch.from_numpy(0.3 * on).cuda()
    out = torch.zeros((1, 4, n, n), dtype=torch.float64, device="cuda")
    for kw in (dict(dt=0.0), dict(steps=0), dict(out_stride=0), dict(out_stride=5), dict(law=2)):
        base = dict(dt=2e-4, steps=4, window=2, law=0, beta=0.017, out_stride=1)
        base.update(kw)
        o = dg.trace_opts(**base)
        with pytest.raises(GtError) as e:
            dg.trace_batch_device(blk_d.data_ptr(), 0, sch_d.data_ptr(), sched.shape[2], l0_d.data_ptr(), 0, 1, o,
                                  out.data_ptr())
        assert e.value.status == 2, kw


def test_trace_batch_n512_warp_rows(b200lib, oracle, tmp_path):
    """n = 512 (m = 1024): the warp-per-row passes with the 32-point register DFT."""
    import ctypes as C
    from paper_2307_12119_b200.api import GreensArrays
    n = 512
    (tmp_path / "stack.txt").write_text(f"n {n}\ndie_edge 0.016\n")
    (tmp_path / "var.txt").write_text("dopant_spread 0\nbeta 0.017\n")
    L = b200lib
    g = C.c_void_p()
    assert L.gt_calibrate(str(tmp_path / "stack.txt").encode(), str(tmp_path / "var.txt").encode(), None, 90.0,
                          C.byref(g), None) == 0, L.gt_last_error()
    maps = {}
    for k in ("f_sp0", "g_sp0"):
        f = C.c_void_p()
        assert L.gt_greens_field(g, k.encode(), C.byref(f)) == 0
        maps[k] = np.ctypeslib.as_array(L.gt_field_data(f), shape=(n, n)).copy()
        L.gt_field_free(f)
    fs = maps["f_sp0"]
    ga = GreensArrays(n=n, pitch=0.016 / n, f_sp0=fs, g_sp0=maps["g_sp0"],
                      phi=float(np.mean(np.concatenate([fs[0], fs[-1], fs[1:-1, 0], fs[1:-1, -1]]))),
                      kappa_inf=float(fs[0, 0]), alpha=L.gt_greens_alpha(g), beta=0.017, mu=L.gt_greens_mu(g),
                      capacitance=L.gt_greens_capacitance(g), rand_scale=1.0)
    L.gt_greens_free(g)
    B, steps, dt, stride, window = 2, 6, 1e-5, 2, 3
    blk, sched, on = _traces(B, steps, n=n, blocks=32, switch_prob=0.3)
    leak0 = 0.3 * on
    ref, st, secs = oracle.trace_leak_batch(ga, blk, sched, leak0, dt, window, law=0, beta=0.017, out_stride=stride)
    assert (st == 0).all()
    for prec, atol in ((1, 1e-8), (0, 1e-3)):
        out, mx = _run_gpu(ga, prec, blk, sched, leak0, dt, window, 0, 0.017, stride)
        err = np.abs(out - ref).max()
        print(f"n=512 prec={prec}: max|dT| {err:.3e} K on peak {ref.max():.2f} K (oracle {secs:.1f} s)")
        assert err <= atol
