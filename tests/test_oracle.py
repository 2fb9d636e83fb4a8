"""Pin the CPU oracle before trusting it (CPU only).

The oracle is the UNCHANGED reference core compiled against FFTW/Eigen subset
shims (oracle/Makefile). These tests check (1) the FFTW shim against numpy's
DFT to 1e-12 (the reference's transform convention, spectral.hpp:12-20),
(2) that the oracle reproduces the committed goldens it generated, and
(3) reference identities SPEC.md lists but the reference never tests.
"""
import ctypes as C
import dataclasses

import numpy as np
import pytest

from conftest import GOLDEN


def _fftw(oracle, x, sign):
    L = C.CDLL(str(oracle.REF_SO))
    L.fftw_plan_dft_2d.restype = C.c_void_p
    L.fftw_plan_dft_2d.argtypes = [C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_int, C.c_uint]
    L.fftw_execute_dft.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
    y = np.ascontiguousarray(x.astype(np.complex128))
    p = L.fftw_plan_dft_2d(y.shape[0], y.shape[1], None, None, sign, 64)
    L.fftw_execute_dft(p, y.ctypes.data, y.ctypes.data)
    return y


@pytest.mark.parametrize("m", [4, 6, 32, 128, 512])
def test_fftw_shim_matches_numpy(oracle, m):
    rng = np.random.default_rng(m)
    x = rng.standard_normal((m, m)) + 1j * rng.standard_normal((m, m))
    fwd = _fftw(oracle, x, -1)
    assert np.abs(fwd - np.fft.fft2(x)).max() <= 1e-12 * np.abs(fwd).max()
    inv = _fftw(oracle, x, +1)  # unnormalised backward
    assert np.abs(inv - np.fft.ifft2(x) * m * m).max() <= 1e-12 * np.abs(inv).max()


def test_fdm_impulse_response_shape(oracle):
    # reference greens.cpp:96-106 invariants: non-negative, peak at the source cell.
    f = oracle.impulse_response(16, 0.016)
    assert f.min() >= 0.0
    assert np.unravel_index(np.argmax(f), f.shape) == (8, 8)


def test_oracle_reproduces_calibration_golden(oracle):
    z = np.load(GOLDEN / "greens_n64.npz")
    g = oracle.calibrate(64, die_edge=0.016, beta=0.017, dopant_spread=0.0, leak_total=84.0,
                         fit_rand_scale=True, fit_transient=True)
    for k in ("f_sp0", "g_sp0", "f_det", "f_rand", "p_var"):
        np.testing.assert_allclose(g[k], z[k], rtol=1e-12, atol=1e-12 * np.abs(z[k]).max())
    for k in ("phi", "kappa_inf", "alpha", "mu", "rand_scale", "capacitance"):
        assert g[k] == pytest.approx(float(z[k]), rel=1e-10)


def test_oracle_reproduces_mc_golden(oracle, greens64):
    m = np.load(GOLDEN / "mc_n64.npz")
    g = dataclasses.replace(greens64, rand_scale=float(m["rand_scale"]))
    t, mx, mean, st, _ = oracle.mc_batch(g, m["p_dyn"], m["var"], leak_frac=float(m["leak_frac"]),
                                         mu_per_sample=1, jobs=2)
    assert (st == 0).all()
    np.testing.assert_allclose(t, m["t_mu_sample"], rtol=0, atol=1e-9)
    np.testing.assert_allclose(mx, m["max_mu_sample"], rtol=1e-12)
    _, mx0, mean0, st0, _ = oracle.mc_batch(g, m["p_dyn"], m["var"], leak_frac=float(m["leak_frac"]),
                                            mu_per_sample=0, jobs=2, want_maps=False)
    np.testing.assert_allclose(mx0, m["max_mu_greens"], rtol=1e-12)


def test_mc_zero_alpha_beta_reduces_to_baseline(oracle, greens64):
    """(alpha, beta) = (0, 0) => F_det == fk (greens.cpp:212; SPEC identity)."""
    m = np.load(GOLDEN / "mc_n64.npz")
    g = dataclasses.replace(greens64, alpha=0.0, beta=0.0, rand_scale=1.0)
    t, _, _, st, _ = oracle.mc_batch(g, m["p_dyn"][:1], m["var"][:1], with_rand=0, jobs=1)
    # linear: doubling the applied map doubles the rise
    t2, _, _, _, _ = oracle.mc_batch(g, 2 * m["p_dyn"][:1].astype(np.float64), m["var"][:1], with_rand=0, jobs=1)
    assert (st == 0).all()
    np.testing.assert_allclose(t2, 2 * t, rtol=1e-10, atol=1e-9)


def test_reference_abi_exports(oracle):
    from paper_2307_12119_b200.api import CORE_SYMBOLS
    L = oracle.ref_lib()
    for s in CORE_SYMBOLS:
        getattr(L, s)
