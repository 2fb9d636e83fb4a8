"""Mode B (north-star leakage fixed point + Kirchhoff transform) on the GPU vs
the fp64 CPU restatement (oracle/restate.cpp ref_fixed_point_batch), which
follows the reference FDM outer loop (fdm.cpp:167-205) with the Green
convolution in place of the CG solve.

fp64: 1e-8 K when both sides stop at the same iteration; fp32: 1e-3 K.
"""
import dataclasses

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu


def _dg(g, prec):
    from paper_2307_12119_b200.api import DeviceGreens
    return DeviceGreens(g, prec)


@pytest.fixture(scope="module")
def golden():
    return np.load(GOLDEN / "mc_n64.npz")


@pytest.mark.parametrize("law,kirchhoff,scale", [(0, 0, 1.0), (0, 1, 0.5), (1, 1, 0.15), (1, 0, 0.25)])
def test_fixed_point_matches_oracle(b200lib, oracle, greens64, golden, law, kirchhoff, scale):
    p = golden["p_dyn"].astype(np.float64) * scale
    v = golden["var"].astype(np.float64)
    kw = dict(leak_frac=0.3, beta=0.017, law=law, kirchhoff=kirchhoff, tol=1e-4, max_iters=80)
    t_ref, it_ref, st_ref, _ = oracle.fixed_point_batch(greens64, p, v, jobs=4, **kw)
    assert (st_ref == 0).all(), st_ref
    for prec, atol in ((1, 1e-8), (0, 1e-3)):
        dg = _dg(greens64, prec)
        kwp = dict(kw)
        if prec == 0 and kirchhoff:
            # fp32 FFT noise (~1e-4 K) times the Kirchhoff slope dT/dtheta = (T/T0)^eta (~3.6 at
            # 850 K) sits above a 1e-4 K stop rule; the fp32 path stops at 5e-4 K.
            kwp["tol"] = 5e-4
            atol = 2e-3
        out, it, st, mx, _ = dg.fp_batch_host(p, v, dg.fp_opts(**kwp))
        assert (st == 0).all(), st
        err = np.abs(out.astype(np.float64) - t_ref).max()
        print(f"law={law} kirchhoff={kirchhoff} prec={prec}: iters {it.tolist()} vs ref {it_ref.tolist()}, "
              f"max|dT|={err:.3e} K, peak {t_ref.max():.1f} K")
        if prec == 1:
            np.testing.assert_array_equal(it, it_ref)
        elif not kirchhoff:
            assert np.abs(it - it_ref).max() <= 3  # fp32 rounding moves the 1e-4 K crossing
        assert err <= atol
        np.testing.assert_allclose(mx, t_ref.reshape(len(p), -1).max(axis=1), atol=atol)


def test_exp_law_runaway_literal_config(b200lib, oracle, greens64, golden):
    """Config 0/1 power with exp(beta dT): no fixed point -> both fail."""
    p = golden["p_dyn"].astype(np.float64)
    v = golden["var"].astype(np.float64)
    kw = dict(leak_frac=0.3, beta=0.017, law=1, kirchhoff=1, tol=1e-4, max_iters=50)
    _, _, st_ref, _ = oracle.fixed_point_batch(greens64, p, v, jobs=4, **kw)
    assert (st_ref != 0).all()
    dg = _dg(greens64, 1)
    _, _, st, _, _ = dg.fp_batch_host(p, v, dg.fp_opts(**kw))
    assert (st != 0).all(), st
    assert ((st & (16 | 32 | 64)) != 0).all()


def test_max_iters_is_convergence_error(b200lib, oracle, greens64, golden):
    p = golden["p_dyn"][:2].astype(np.float64)
    v = golden["var"][:2].astype(np.float64)
    kw = dict(leak_frac=0.3, beta=0.017, law=0, kirchhoff=0, tol=1e-4, max_iters=3)
    _, it_ref, st_ref, _ = oracle.fixed_point_batch(greens64, p, v, jobs=2, **kw)
    assert (st_ref == 3).all() and (it_ref == 3).all()
    dg = _dg(greens64, 1)
    _, it, st, _, _ = dg.fp_batch_host(p, v, dg.fp_opts(**kw))
    assert (st == 32).all() and (it == 3).all()


def test_linear_uniform_reduces_to_closed_form(b200lib, greens64):
    """Linear law, alpha = 0, uniform leakage: the fixed point is the geometric
    series of the closed form 1/(1 - mu beta F(f_sp0)) (greens.cpp:212). The
    die-domain iteration re-mirrors each iterate, so it differs from the torus
    closed form only through the one-cell kernel asymmetry."""
    g = dataclasses.replace(greens64, alpha=0.0, rand_scale=1.0)
    n = g.n
    p = np.full((1, n, n), 60.0 / (n * n))
    v = np.ones((1, n, n))
    dg = _dg(g, 1)
    tb, it, st, _, _ = dg.fp_batch_host(p, v, dg.fp_opts(law=0, kirchhoff=0, beta=0.017, tol=1e-9, max_iters=200))
    assert st[0] == 0
    ta, _, _, sa, _ = dg.mc_batch_host(p, v, dg.opts(leak_frac=0.3, mu_per_sample=1, with_rand=0))
    assert sa[0] == 0
    gap = np.abs(tb - ta).max()
    print(f"die-domain fixed point vs closed form: {gap:.3e} K on peak {ta.max():.2f} K after {it[0]} iterations")
    assert gap <= 2e-3 * ta.max()
