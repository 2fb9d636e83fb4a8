"""The FDM reference solver entries (gt_oracle_steady / gt_oracle_transient) on
the device (fdm.cu: matrix-free 3-layer network, Jacobi-PCG with Eigen's stopping
rule) against the SAME entries of the reference library (oracle/_ref, Eigen-shim
CG / LDLT), through the identical C ABI on the identical stack / variation files.
The CG stops at a 1e-9 relative residual on both sides: agreement to ~1e-6 K."""
import ctypes as C
import dataclasses

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ATOL = 2e-6


def _field(L, arr, pitch, unit=b"watts"):
    f = C.c_void_p()
    assert L.gt_field_create(arr.shape[0], pitch, unit, C.byref(f)) == 0
    np.ctypeslib.as_array(L.gt_field_data(f), shape=arr.shape)[...] = arr
    return f


def _map(L, f, n):
    return np.ctypeslib.as_array(L.gt_field_data(f), shape=(n, n)).copy()


@pytest.fixture(scope="module")
def setup(tmp_path_factory):
    from paper_2307_12119_b200 import inputs
    d = tmp_path_factory.mktemp("fdm")
    n = 32
    (d / "stack.txt").write_text(f"n {n}\ndie_edge 0.016\n")
    (d / "var.txt").write_text("dopant_spread 0.05\nbeta 0.017\nseed 7\n")
    cfg = dataclasses.replace(inputs.CONFIGS["cfg0"], n=n, blocks=8)
    p = inputs.power_map(cfg, 0) * 0.3
    leak = 0.3 * p
    return d, n, 0.016 / n, p, leak


@pytest.mark.parametrize("use_var,tdl,tdc", [(False, 0, 0), (True, 1, 0), (True, 1, 1), (True, 0, 1)])
def test_oracle_steady_matches_reference(b200lib, oracle, setup, use_var, tdl, tdc):
    d, n, pitch, p, leak = setup
    res = []
    for L in (b200lib, oracle.ref_lib()):
        pf, lf = _field(L, p, pitch), _field(L, leak, pitch)
        out, it = C.c_void_p(), C.c_int()
        st = L.gt_oracle_steady(str(d / "stack.txt").encode(), str(d / "var.txt").encode() if use_var else None,
                                pf, lf if (tdl or use_var) else None, tdl, tdc, C.byref(out), C.byref(it))
        assert st == 0, L.gt_last_error()
        res.append((_map(L, out, n), it.value))
        for f in (pf, lf, out):
            L.gt_field_free(f)
    err = np.abs(res[0][0] - res[1][0]).max()
    print(f"oracle steady var={use_var} tdl={tdl} tdc={tdc}: iters {res[0][1]} vs {res[1][1]}, "
          f"max|dT| {err:.2e} K on peak {res[1][0].max():.2f} K")
    assert res[0][1] == res[1][1]
    assert err <= ATOL


def test_oracle_transient_matches_reference(b200lib, oracle, setup):
    d, n, pitch, p, leak = setup
    times = np.array([2e-4, 5e-4, 1.5e-3])
    res = []
    for L in (b200lib, oracle.ref_lib()):
        pf, lf = _field(L, p, pitch), _field(L, leak, pitch)
        r = C.c_void_p()
        st = L.gt_oracle_transient(str(d / "stack.txt").encode(), str(d / "var.txt").encode(), pf, lf, 1,
                                   times.ctypes.data_as(C.POINTER(C.c_double)), len(times), 1e-4, C.byref(r))
        assert st == 0, L.gt_last_error()
        maps = []
        for i in range(L.gt_result_count(r)):
            f = C.c_void_p()
            assert L.gt_result_map(r, i, C.byref(f)) == 0
            maps.append(_map(L, f, n))
            L.gt_field_free(f)
        res.append(np.array(maps))
        for f in (pf, lf):
            L.gt_field_free(f)
    err = np.abs(res[0] - res[1]).max()
    print(f"oracle transient: max|dT| {err:.2e} K on peak {res[1].max():.3f} K")
    assert err <= ATOL


def test_oracle_error_behaviour_matches_reference(b200lib, oracle, setup):
    """Negative power -> config error; temp-dependent leakage without a nominal map is
    ignored (reference oracle_setup only enables it with a leakage baseline)."""
    d, n, pitch, p, leak = setup
    for arr, tdl, want in ((-p, 0, 2), (p, 1, 0)):
        got = []
        for L in (b200lib, oracle.ref_lib()):
            pf = _field(L, arr, pitch)
            out, it = C.c_void_p(), C.c_int()
            got.append(L.gt_oracle_steady(str(d / "stack.txt").encode(), None, pf, None, tdl, 0, C.byref(out),
                                          C.byref(it)))
            L.gt_field_free(pf)
        assert got == [want, want], got
