"""Mode-A Monte-Carlo batch on the GPU vs the CPU oracle (the reference's own
run_one arithmetic, solver.cpp:353-374) through the C ABI.

Tolerances: fp64 device path vs fp64 reference: 1e-8 K absolute (FFT
algorithm differences only). fp32 device path: the north-star bar of
1e-3 K maximum absolute error (BASELINE.json).
"""
import dataclasses

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu

FP64_ATOL = 1e-8
FP32_ATOL = 1e-3


def _dg(g, prec):
    from paper_2307_12119_b200.api import DeviceGreens
    return DeviceGreens(g, prec)


@pytest.fixture(scope="module")
def golden():
    return np.load(GOLDEN / "mc_n64.npz")


@pytest.fixture(scope="module")
def g64(greens64, golden):
    return dataclasses.replace(greens64, rand_scale=float(golden["rand_scale"]))


@pytest.mark.parametrize("prec,atol", [(1, FP64_ATOL), (0, FP32_ATOL)])
def test_mc_matches_golden(b200lib, g64, golden, prec, atol):
    dg = _dg(g64, prec)
    out, mx, mean, st, _ = dg.mc_batch_host(golden["p_dyn"], golden["var"], dg.opts(mu_per_sample=1))
    assert (st == 0).all(), st
    err = np.abs(out.astype(np.float64) - golden["t_mu_sample"]).max()
    print(f"prec={prec} max|dT|={err:.3e} K on peak {golden['max_mu_sample'].max():.1f} K")
    assert err <= atol
    np.testing.assert_allclose(mx, golden["max_mu_sample"], rtol=0, atol=atol)
    np.testing.assert_allclose(mean, golden["mean_mu_sample"], rtol=0, atol=atol)


@pytest.mark.parametrize("prec,atol", [(1, FP64_ATOL), (0, FP32_ATOL)])
def test_mc_greens_mu_mode(b200lib, g64, golden, prec, atol):
    """mu_per_sample = 0: closed forms at the GreensSet mu (reference monte_carlo)."""
    dg = _dg(g64, prec)
    _, mx, mean, st, _ = dg.mc_batch_host(golden["p_dyn"], golden["var"], dg.opts(mu_per_sample=0),
                                          want_maps=False)
    assert (st == 0).all()
    np.testing.assert_allclose(mx, golden["max_mu_greens"], rtol=0, atol=atol)
    np.testing.assert_allclose(mean, golden["mean_mu_greens"], rtol=0, atol=atol)


@pytest.mark.parametrize("n", [16, 32, 128])
def test_mc_live_oracle_sizes(b200lib, oracle, n):
    """Other grid sizes: reference calibrate() at n, fresh seeded inputs, live oracle."""
    from paper_2307_12119_b200 import inputs
    from paper_2307_12119_b200.api import GreensArrays
    d = oracle.calibrate(n, die_edge=0.016, beta=0.017, leak_total=84.0, fit_rand_scale=False)
    g = GreensArrays(**{k: d[k] for k in ("n", "pitch", "f_sp0", "g_sp0", "phi", "kappa_inf", "alpha", "beta",
                                           "mu")}, rand_scale=1.0)
    cfg = dataclasses.replace(inputs.CONFIGS["cfg1"], n=n, blocks=min(32, n * n // 16), base_seed=77 + n)
    B = 5
    p = inputs.power_batch(cfg, 0, B, np.float64)
    v = inputs.variation_batch(cfg, 0, B).numpy().astype(np.float64)
    t_ref, mx_ref, _, st_ref, _ = oracle.mc_batch(g, p, v, jobs=4)
    assert (st_ref == 0).all()
    dg = _dg(g, 1)
    out, mx, _, st, _ = dg.mc_batch_host(p, v, dg.opts())
    assert (st == 0).all()
    assert np.abs(out - t_ref).max() <= FP64_ATOL


def test_mc_config1_grid_fp32(b200lib, oracle, greens256):
    """The headline grid (n = 256, config-1 generator) in fp32 against the fp64 reference."""
    from paper_2307_12119_b200 import inputs
    cfg = inputs.CONFIGS["cfg1"]
    B = 6
    p = inputs.power_batch(cfg, 0, B, np.float32)
    v = inputs.variation_batch(cfg, 0, B).numpy().astype(np.float32)
    t_ref, mx_ref, _, st_ref, _ = oracle.mc_batch(greens256, p, v, jobs=8)
    assert (st_ref == 0).all()
    for prec, atol in ((0, FP32_ATOL), (1, FP64_ATOL)):
        dg = _dg(greens256, prec)
        out, mx, _, st, _ = dg.mc_batch_host(p, v, dg.opts())
        assert (st == 0).all()
        err = np.abs(out.astype(np.float64) - t_ref).max()
        print(f"n=256 prec={prec} max|dT|={err:.3e} K (peak {t_ref.max():.1f} K)")
        assert err <= atol


@pytest.mark.parametrize("mu_per_sample", [0, 1])
def test_mc_config1_grid_maps_both_mu_modes(b200lib, oracle, greens256, mu_per_sample):
    """Maps at the headline grid for both closed-form mu semantics: 0 = the reference
    monte_carlo (F_det and F_rand at gs.mu, solver.cpp:350-351,361: the fixed-mu
    table kernel), 1 = per-sample mean leakage. fp32 <= 1e-3 K, fp64 <= 1e-8 K."""
    from paper_2307_12119_b200 import inputs
    cfg = inputs.CONFIGS["cfg1"]
    B = 8
    p = inputs.power_batch(cfg, 100, B, np.float32)
    v = inputs.variation_batch(cfg, 100, B).numpy().astype(np.float32)
    t_ref, mx_ref, mean_ref, st_ref, _ = oracle.mc_batch(greens256, p, v, mu_per_sample=mu_per_sample, jobs=8)
    assert (st_ref == 0).all()
    for prec, atol in ((0, FP32_ATOL), (1, FP64_ATOL)):
        dg = _dg(greens256, prec)
        out, mx, mean, st, _ = dg.mc_batch_host(p, v, dg.opts(mu_per_sample=mu_per_sample))
        assert (st == 0).all()
        err = np.abs(out.astype(np.float64) - t_ref).max()
        print(f"n=256 mu_per_sample={mu_per_sample} prec={prec} max|dT|={err:.3e} K (peak {t_ref.max():.1f} K)")
        assert err <= atol
        np.testing.assert_allclose(mx, mx_ref, rtol=0, atol=atol)
        np.testing.assert_allclose(mean, mean_ref, rtol=0, atol=atol)


def test_mc_sample_status_isolated(b200lib, g64, golden):
    """A bad sample is flagged (check_power / exponent cap) without touching its neighbours."""
    p = golden["p_dyn"].astype(np.float64).copy()
    v = golden["var"].astype(np.float64).copy()
    p[1, 3, 3] = -1.0        # ConfigError in the reference (solver.cpp:63-70)
    v[2, 0, 0] = np.exp(7.0)  # |ln var| > 6: ValidationError (variation.cpp:173-178)
    dg = _dg(g64, 1)
    out, mx, _, st, _ = dg.mc_batch_host(p, v, dg.opts())
    assert st[0] == 0 and st[3] == 0
    assert st[1] & 1 and st[2] & 2
    np.testing.assert_allclose(out[0], golden["t_mu_sample"][0], atol=FP64_ATOL)
    np.testing.assert_allclose(out[3], golden["t_mu_sample"][3], atol=FP64_ATOL)


def test_mc_runaway_flag(b200lib, oracle, g64, golden):
    """Leakage feedback gain exactly at unity at DC -> the deterministic denominator
    1 - mu beta F(f_sp0) collapses: RunawayError in the reference (greens.cpp:32-39)."""
    fk0 = float(np.sum(g64.f_sp0))  # fk[0,0] = sum(f_sp0 - phi) + phi m^2/4 (greens.cpp:194-201)
    g = dataclasses.replace(g64, beta=1.0 / (g64.mu * fk0))
    p, v = golden["p_dyn"][:2], golden["var"][:2]
    _, _, _, st_ref, _ = oracle.mc_batch(g, p, v, mu_per_sample=0, jobs=2, want_maps=False)
    assert (st_ref == 3).all()
    for prec in (0, 1):
        dg = _dg(g, prec)
        _, _, _, st, _ = dg.mc_batch_host(p, v, dg.opts(mu_per_sample=0), want_maps=False)
        assert ((st & 4) != 0).all(), st


def test_mc_chunking_is_invisible(b200lib, g64, golden):
    p = np.concatenate([golden["p_dyn"]] * 3).astype(np.float32)
    v = np.concatenate([golden["var"]] * 3).astype(np.float32)
    dg = _dg(g64, 0)
    a = dg.mc_batch_host(p, v, dg.opts(chunk=5))
    b = dg.mc_batch_host(p, v, dg.opts(chunk=12))
    np.testing.assert_array_equal(a[0], b[0])
    np.testing.assert_array_equal(a[1], b[1])


def test_mc_device_resident_equals_host_path(b200lib, g64, golden):
    import torch
    from paper_2307_12119_b200.api import SAMPLE_STATS_DTYPE
    dg = _dg(g64, 0)
    p = torch.from_numpy(golden["p_dyn"]).cuda()
    v = torch.from_numpy(golden["var"]).cuda()
    out = torch.empty_like(p)
    B = p.shape[0]
    stats = torch.zeros(B * SAMPLE_STATS_DTYPE.itemsize, dtype=torch.uint8, device="cuda")
    dg.mc_batch_device(p.data_ptr(), v.data_ptr(), B, dg.opts(), out.data_ptr(), stats.data_ptr(),
                       torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    st = np.frombuffer(stats.cpu().numpy().tobytes(), dtype=SAMPLE_STATS_DTYPE)
    h_out, h_mx, _, _, _ = dg.mc_batch_host(golden["p_dyn"], golden["var"], dg.opts())
    np.testing.assert_array_equal(out.cpu().numpy(), h_out)
    np.testing.assert_array_equal(st["max_rise"], h_mx)


def test_mc_calls_on_different_streams_are_ordered(b200lib, g64, golden):
    """Two device calls on one handle, enqueued back to back on different streams
    without a host sync, share the handle's scratch: the second call's stream
    waits for the first call's work, so both results equal the sequential ones."""
    import torch
    from paper_2307_12119_b200.api import SAMPLE_STATS_DTYPE
    dg = _dg(g64, 0)
    p = torch.from_numpy(golden["p_dyn"]).cuda()
    v = torch.from_numpy(golden["var"]).cuda()
    B = p.shape[0]
    p2 = (p * 0.5).contiguous()
    ref1, _, _, _, _ = dg.mc_batch_host(golden["p_dyn"], golden["var"], dg.opts())
    ref2, _, _, _, _ = dg.mc_batch_host(p2.cpu().numpy(), golden["var"], dg.opts())
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    o1, o2 = torch.empty_like(p), torch.empty_like(p)
    st1 = torch.zeros(B * SAMPLE_STATS_DTYPE.itemsize, dtype=torch.uint8, device="cuda")
    st2 = torch.zeros_like(st1)
    torch.cuda.synchronize()
    for _ in range(3):
        dg.mc_batch_device(p.data_ptr(), v.data_ptr(), B, dg.opts(), o1.data_ptr(), st1.data_ptr(), s1.cuda_stream)
        dg.mc_batch_device(p2.data_ptr(), v.data_ptr(), B, dg.opts(), o2.data_ptr(), st2.data_ptr(), s2.cuda_stream)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(o1.cpu().numpy(), ref1)
        np.testing.assert_array_equal(o2.cpu().numpy(), ref2)
        st1.zero_()
        st2.zero_()


def test_mc_unaligned_inputs_take_the_direct_load_path(b200lib, g64, golden):
    """Row passes stage their input rows with 16-byte TMA bulk copies when the maps
    are 16-byte aligned; maps that start 4 bytes into a buffer take the direct-load
    kernels instead. Both paths do the same arithmetic: results are bit-identical."""
    import torch
    from paper_2307_12119_b200.api import SAMPLE_STATS_DTYPE
    dg = _dg(g64, 0)
    B, n = golden["p_dyn"].shape[0], golden["p_dyn"].shape[1]
    pa = torch.from_numpy(golden["p_dyn"]).cuda()
    va = torch.from_numpy(golden["var"]).cuda()
    pb = torch.zeros(B * n * n + 1, dtype=torch.float32, device="cuda")
    vb = torch.zeros_like(pb)
    pb[1:] = pa.reshape(-1)
    vb[1:] = va.reshape(-1)
    outs = []
    for p_ptr, v_ptr in ((pa.data_ptr(), va.data_ptr()), (pb.data_ptr() + 4, vb.data_ptr() + 4)):
        assert (p_ptr % 16 == 0) == (p_ptr == pa.data_ptr())
        out = torch.empty_like(pa)
        stats = torch.zeros(B * SAMPLE_STATS_DTYPE.itemsize, dtype=torch.uint8, device="cuda")
        dg.mc_batch_device(p_ptr, v_ptr, B, dg.opts(), out.data_ptr(), stats.data_ptr(),
                           torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        st = np.frombuffer(stats.cpu().numpy().tobytes(), dtype=SAMPLE_STATS_DTYPE)
        assert (st["status"] == 0).all()
        outs.append((out.cpu().numpy(), st["max_rise"].copy(), st["mean_rise"].copy()))
    for a, b in zip(outs[0], outs[1]):
        np.testing.assert_array_equal(a, b)
    err = np.abs(outs[0][0].astype(np.float64) - golden["t_mu_sample"]).max()
    assert err <= FP32_ATOL


def test_profile_modes(b200lib, g64, golden):
    """gt_profile_begin_mode: mode 0 times the three passes, mode 1 the column pass
    only (pass_ms[0] = pass_ms[2] = 0); both count the same launches and calls."""
    import torch
    from paper_2307_12119_b200.api import SAMPLE_STATS_DTYPE
    dg = _dg(g64, 0)
    p = torch.from_numpy(golden["p_dyn"]).cuda()
    v = torch.from_numpy(golden["var"]).cuda()
    B = p.shape[0]
    out = torch.empty_like(p)
    stats = torch.zeros(B * SAMPLE_STATS_DTYPE.itemsize, dtype=torch.uint8, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    res = {}
    for mode in (0, 1):
        dg.profile_begin(mode)
        for _ in range(3):
            dg.mc_batch_device(p.data_ptr(), v.data_ptr(), B, dg.opts(), out.data_ptr(), stats.data_ptr(), s)
        res[mode] = dg.profile_end()
    (ms0, k0, c0), (ms1, k1, c1) = res[0], res[1]
    assert all(x > 0 for x in ms0[:3]) and abs(ms0[3] - sum(ms0[:3])) < 1e-9
    assert ms1[0] == 0 and ms1[2] == 0 and ms1[1] > 0
    assert (k0, c0) == (k1, c1) and c0 == 3
    with pytest.raises(Exception):
        dg.profile_begin(2)


def _cfg1_pairs(idx):
    """Config-1 pairs by global sample index, generated as bench.py does (fp32 on the device)."""
    import torch
    from paper_2307_12119_b200 import inputs
    P, V = inputs.mc_inputs(inputs.CONFIGS["cfg1"], 0, max(idx) + 1, device="cuda", torch_dtype=torch.float32)
    sel = torch.tensor(idx, device="cuda")
    return P[sel].cpu().numpy(), V[sel].cpu().numpy()


@pytest.mark.parametrize("mu_per_sample", [0, 1])
def test_mc_fp64_resolve_of_ill_conditioned_pairs(b200lib, greens256, mu_per_sample):
    """'fp32 with fp64 residual check' (BASELINE config 1): config-1 pairs whose random_greens
    denominator comes close to singular (pairs 25, 63, 114, 454 of the bench batch: fp32 error up
    to 1.3e-2 K without the check) are re-solved in fp64 on the device; every pair then meets
    1e-3 K against the fp64 path, and the re-solved ones are marked by a negative max_rden2."""
    from paper_2307_12119_b200.api import SAMPLE_STATS_DTYPE  # noqa: F401
    idx = [25, 63, 114, 454, 0, 1, 2, 3, 270, 5, 6, 7, 8, 9, 10, 11]
    p, v = _cfg1_pairs(idx)
    d64 = _dg(greens256, 1)
    ref = d64.mc_batch_host(p.astype(np.float64), v.astype(np.float64), d64.opts(mu_per_sample=mu_per_sample))
    d32 = _dg(greens256, 0)
    raw = d32.mc_batch_host(p, v, d32.opts(mu_per_sample=mu_per_sample, fp64_check=-1.0))
    chk = d32.mc_batch_host(p, v, d32.opts(mu_per_sample=mu_per_sample))
    e_raw = np.abs(raw[0].astype(np.float64) - ref[0]).reshape(len(idx), -1).max(1)
    e_chk = np.abs(chk[0].astype(np.float64) - ref[0]).reshape(len(idx), -1).max(1)
    print(f"mu_per_sample={mu_per_sample}: fp32 max err without check {e_raw.max():.3e} K, with {e_chk.max():.3e} K")
    assert e_raw.max() > FP32_ATOL  # the check is needed on these pairs
    assert (chk[3] == 0).all()
    assert e_chk.max() <= FP32_ATOL
    np.testing.assert_allclose(chk[1], ref[1], rtol=0, atol=FP32_ATOL)


def test_mc_fp64_resolve_capacity(b200lib, g64, golden):
    """Threshold below every pair: all pairs qualify, the first batch/16 (min 8) are re-solved
    in fp64 (marked by max_rden2 < 0, results = the fp64 path) and the rest carry
    GT_SAMPLE_ILLCOND (128) with their fp32 results."""
    import torch
    from paper_2307_12119_b200.api import SAMPLE_STATS_DTYPE
    p = np.concatenate([golden["p_dyn"]] * 3)
    v = np.concatenate([golden["var"]] * 3)
    B = p.shape[0]
    d64 = _dg(g64, 1)
    ref = d64.mc_batch_host(p.astype(np.float64), v.astype(np.float64), d64.opts(mu_per_sample=0))[0]
    d32 = _dg(g64, 0)
    P, V = torch.from_numpy(p.astype(np.float32)).cuda(), torch.from_numpy(v.astype(np.float32)).cuda()
    out = torch.empty_like(P)
    stats = torch.zeros(B * SAMPLE_STATS_DTYPE.itemsize, dtype=torch.uint8, device="cuda")
    d32.mc_batch_device(P.data_ptr(), V.data_ptr(), B, d32.opts(mu_per_sample=0, fp64_check=1e-30), out.data_ptr(),
                        stats.data_ptr(), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    st = np.frombuffer(stats.cpu().numpy().tobytes(), dtype=SAMPLE_STATS_DTYPE)
    resolved = st["max_rden2"] < 0
    assert resolved.sum() == 8 and ((st["status"] == 128) == ~resolved).all()
    o = out.double().cpu().numpy()
    np.testing.assert_allclose(o[resolved], ref[resolved].astype(np.float32).astype(np.float64), rtol=0, atol=1e-9)
    assert np.abs(o[~resolved] - ref[~resolved]).max() <= FP32_ATOL
