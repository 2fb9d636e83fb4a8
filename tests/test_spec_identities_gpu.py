"""Known-answer identities of the reference's operation spec (the
SPEC.md properties the reference lists but never tests), run on the GPU path:

* (alpha, beta) = 0 reduces the deterministic closed form to the baseline
  kernel, F_det = fk (greens.cpp:203-216), so a leakage-free mode-A solve is
  exactly crop(IFFT2(fk . FFT2(mirror(P)))) -- checked against numpy fp64;
* linearity of the deterministic path in the power map;
* p_var = 0 (uniform leakage) makes the shift-variant term vanish;
* Monte-Carlo results are byte-deterministic run to run;
* step response: t = 0 gives 0 and t -> infinity gives the steady map;
* a constant power trace converges to the steady map.
"""
import ctypes as C
import dataclasses

import numpy as np
import pytest

from slab_numpy_ops import baseline_fk

pytestmark = pytest.mark.gpu


def _det0(greens64):
    return dataclasses.replace(greens64, alpha=0.0, beta=0.0)


def _numpy_det(g, P):
    n = P.shape[0]
    m = 2 * n
    i = np.arange(m)
    mi = np.where(i < n, i, m - 1 - i)
    fk = baseline_fk(g.f_sp0, g.phi)
    T = np.fft.ifft2(fk * np.fft.fft2(P[np.ix_(mi, mi)])).real[:n, :n]
    return np.maximum(T, 0.0)


def _maps(n, k, seed):
    rng = np.random.default_rng(seed)
    return rng.uniform(0.0, 0.05, size=(k, n, n))


def test_alpha_beta_zero_is_the_baseline_convolution(b200lib, greens64):
    from paper_2307_12119_b200.api import DeviceGreens
    g = _det0(greens64)
    P = _maps(64, 3, 1)
    V = np.ones_like(P)
    dg = DeviceGreens(g, 1)
    out, _, _, st, _ = dg.mc_batch_host(P, V, dg.opts(leak_frac=0.0, with_rand=0))
    assert (st == 0).all()
    for k in range(P.shape[0]):
        ref = _numpy_det(g, P[k])
        err = np.abs(out[k] - ref).max() / ref.max()
        assert err <= 1e-10, err


def test_deterministic_path_is_linear(b200lib, greens64):
    from paper_2307_12119_b200.api import DeviceGreens
    g = _det0(greens64)
    P = _maps(64, 2, 2)
    mix = P[0] + 2.5 * P[1]
    dg = DeviceGreens(g, 1)
    out, _, _, st, _ = dg.mc_batch_host(np.stack([P[0], P[1], mix]), np.ones((3, 64, 64)),
                                        dg.opts(leak_frac=0.0, with_rand=0))
    assert (st == 0).all()
    lin = out[0] + 2.5 * out[1]
    assert np.abs(out[2] - lin).max() <= 1e-11 * lin.max()


@pytest.mark.parametrize("prec", [1, 0])
def test_uniform_leakage_has_no_shift_variant_term(b200lib, greens64, prec):
    from paper_2307_12119_b200.api import DeviceGreens
    P = np.full((2, 64, 64), 0.02)
    V = np.ones_like(P)
    dg = DeviceGreens(greens64, prec)
    dt = np.float64 if prec else np.float32
    on, _, _, s1, _ = dg.mc_batch_host(P.astype(dt), V.astype(dt), dg.opts(with_rand=1))
    off, _, _, s0, _ = dg.mc_batch_host(P.astype(dt), V.astype(dt), dg.opts(with_rand=0))
    assert (s1 == 0).all() and (s0 == 0).all()
    np.testing.assert_array_equal(on, off)


def test_monte_carlo_is_byte_deterministic(b200lib, greens64):
    from paper_2307_12119_b200 import inputs
    from paper_2307_12119_b200.api import DeviceGreens
    cfg = dataclasses.replace(inputs.CONFIGS["cfg1"], n=64)
    P = inputs.power_batch(cfg, 0, 8, np.float32)
    V = inputs.variation_batch(cfg, 0, 8).numpy().astype(np.float32)
    dg = DeviceGreens(greens64, 0)
    a = dg.mc_batch_host(P, V, dg.opts())
    b = dg.mc_batch_host(P, V, dg.opts())
    for x, y in zip(a[:4], b[:4]):
        assert np.asarray(x).tobytes() == np.asarray(y).tobytes()


def _field(L, arr, pitch):
    f = C.c_void_p()
    assert L.gt_field_create(arr.shape[0], pitch, b"watts", C.byref(f)) == 0
    np.ctypeslib.as_array(L.gt_field_data(f), shape=arr.shape)[...] = arr
    return f


def _map(L, f, n):
    return np.ctypeslib.as_array(L.gt_field_data(f), shape=(n, n)).copy()


@pytest.fixture(scope="module")
def handle(b200lib, greens64):
    g = greens64.to_handle(b200lib)
    yield g
    b200lib.gt_greens_free(g)


def _steady(L, g, P, pitch):
    out = C.c_void_p()
    assert L.gt_solve_steady(g, _field(L, P, pitch), 1, C.byref(out), None) == 0, L.gt_last_error()
    return _map(L, out, P.shape[0])


def test_step_response_limits(b200lib, greens64, handle):
    L = b200lib
    P = _maps(64, 1, 3)[0]
    steady = _steady(L, handle, P, greens64.pitch)
    times = np.array([0.0, 50.0])
    r = C.c_void_p()
    assert L.gt_solve_step(handle, _field(L, P, greens64.pitch), times.ctypes.data_as(C.POINTER(C.c_double)), 2, 1,
                           C.byref(r), None) == 0, L.gt_last_error()
    maps = []
    for i in range(2):
        f = C.c_void_p()
        assert L.gt_result_map(r, i, C.byref(f)) == 0
        maps.append(_map(L, f, 64))
    assert np.abs(maps[0]).max() == 0.0
    assert np.abs(maps[1] - steady).max() <= 1e-9 * steady.max()


def test_constant_trace_converges_to_steady(b200lib, greens64, handle):
    L = b200lib
    P = _maps(64, 1, 4)[0]
    steady = _steady(L, handle, P, greens64.pitch)
    tr = C.c_void_p()
    assert L.gt_trace_create(C.c_double(0.05), C.byref(tr)) == 0
    for _ in range(60):
        assert L.gt_trace_push(tr, _field(L, P, greens64.pitch)) == 0
    r = C.c_void_p()
    assert L.gt_solve_trace(handle, tr, 0, 1, C.byref(r), None) == 0, L.gt_last_error()
    f = C.c_void_p()
    assert L.gt_result_map(r, L.gt_result_count(r) - 1, C.byref(f)) == 0
    last = _map(L, f, 64)
    assert np.abs(last - steady).max() <= 1e-6 * steady.max()
