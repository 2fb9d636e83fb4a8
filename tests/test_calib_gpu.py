"""Device calibration (gt_calibrate: modal kernel producer + closed forms +
capacitance fit) and the reference-API Monte Carlo (gt_monte_carlo) against
the SAME entries of the reference library on identical files.

The reference measures f_sp0 with its FDM network (CG to a 1e-9 relative
residual for n > 16); the device evaluates the exact modal solution of that
network, so maps agree to the CG tolerance, not to rounding.
"""
import csv
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _write(path, text):
    path.write_text(text)
    return str(path).encode()


def _field_arr(L, f, n):
    return np.ctypeslib.as_array(L.gt_field_data(f), shape=(n, n)).copy()


def _greens_maps(L, g, n):
    out = {}
    for k in ("f_sp0", "g_sp0", "f_det", "f_rand", "p_var"):
        f = C.c_void_p()
        assert L.gt_greens_field(g, k.encode(), C.byref(f)) == 0
        out[k] = _field_arr(L, f, n)
        L.gt_field_free(f)
    return out


@pytest.mark.parametrize("n", [32, 64])
def test_calibrate_matches_reference(b200lib, oracle, tmp_path, n):
    stack = _write(tmp_path / "stack.txt", f"n {n}\ndie_edge 0.016\n")
    var = _write(tmp_path / "var.txt", "dopant_spread 0\nbeta 0.017\n")
    res = []
    for L in (b200lib, oracle.ref_lib()):
        g = C.c_void_p()
        ms = C.c_double()
        assert L.gt_calibrate(stack, var, None, 84.0, C.byref(g), C.byref(ms)) == 0, L.gt_last_error()
        res.append((L, g))
    (Lb, gb), (Lr, gr) = res
    mb, mr = _greens_maps(Lb, gb, n), _greens_maps(Lr, gr, n)
    for k in ("f_sp0", "g_sp0"):
        rel = np.abs(mb[k] - mr[k]).max() / np.abs(mr[k]).max()
        print(f"n={n} {k}: max rel diff {rel:.2e}")
        assert rel <= 1e-7
    for getter in ("gt_greens_alpha", "gt_greens_mu", "gt_greens_kappa_inf", "gt_greens_beta"):
        a, b = getattr(Lb, getter)(gb), getattr(Lr, getter)(gr)
        assert a == pytest.approx(b, rel=1e-6), getter
    np.testing.assert_allclose(mb["p_var"], mr["p_var"], rtol=0, atol=1e-12 * np.abs(mr["p_var"]).max() + 1e-15)
    for k in ("f_det", "f_rand"):
        rel = np.abs(mb[k] - mr[k]).max() / np.abs(mr[k]).max()
        print(f"n={n} {k}: max rel diff {rel:.2e}")
        assert rel <= 1e-5
    cb, cr = Lb.gt_greens_capacitance(gb), Lr.gt_greens_capacitance(gr)
    print(f"n={n} capacitance {cb:.6e} vs reference {cr:.6e}")
    assert cb == pytest.approx(cr, rel=1e-4)
    _check_rand_scale(tmp_path, Lb, gb, Lr, gr, n)


def _rand_scale(L, g, d):
    L.gt_greens_save(g, str(d).encode())
    for line in (d / "calibration.txt").read_text().splitlines() + (d / "manifest.txt").read_text().splitlines():
        if line.startswith("rand_scale"):
            return float(line.split()[1])
    raise AssertionError("rand_scale not saved")


def _check_rand_scale(tmp_path, Lb, gb, Lr, gr, n):
    rb, rr = _rand_scale(Lb, gb, tmp_path / "sb"), _rand_scale(Lr, gr, tmp_path / "sr")
    print(f"n={n} rand_scale {rb:.6f} vs reference {rr:.6f}")
    assert rb == pytest.approx(rr, rel=1e-5, abs=1e-6)
    # the 100-map transient tensor (greens.cpp:427-442), as saved by both libraries
    tb = sorted((tmp_path / "sb").glob("tran_*.map"))
    tr = sorted((tmp_path / "sr").glob("tran_*.map"))
    assert len(tb) == len(tr) == 100
    worst = 0.0
    for a, b in zip(tb[::9], tr[::9]):
        ma = np.loadtxt(a, skiprows=1)
        mb = np.loadtxt(b, skiprows=1)
        worst = max(worst, np.abs(ma - mb).max() / np.abs(mb).max())
    print(f"n={n} tran tensor max rel diff {worst:.2e}")
    assert worst <= 1e-5


def test_calibrate_per_cell_conductivity_matches_reference(b200lib, oracle, tmp_path):
    """dopant_spread > 0: f_sp0 and the capacitance target come from the device FDM network
    with the reference's own per-cell conductivity draws."""
    n = 32
    stack = _write(tmp_path / "stack.txt", f"n {n}\ndie_edge 0.016\n")
    var = _write(tmp_path / "var.txt", "dopant_spread 0.05\nbeta 0.017\nseed 3\n")
    res = []
    for L in (b200lib, oracle.ref_lib()):
        g = C.c_void_p()
        assert L.gt_calibrate(stack, var, None, 84.0, C.byref(g), None) == 0, L.gt_last_error()
        res.append((L, g))
    (Lb, gb), (Lr, gr) = res
    mb, mr = _greens_maps(Lb, gb, n), _greens_maps(Lr, gr, n)
    for k in ("f_sp0", "f_det", "f_rand"):
        rel = np.abs(mb[k] - mr[k]).max() / np.abs(mr[k]).max()
        print(f"per-cell k {k}: max rel diff {rel:.2e}")
        assert rel <= 1e-6
    cb, cr = Lb.gt_greens_capacitance(gb), Lr.gt_greens_capacitance(gr)
    print(f"per-cell k capacitance {cb:.6e} vs reference {cr:.6e}")
    assert cb == pytest.approx(cr, rel=1e-4)
    _check_rand_scale(tmp_path, Lb, gb, Lr, gr, n)


@pytest.mark.parametrize("seed_chunk", [None, "4"])
def test_monte_carlo_matches_reference(b200lib, oracle, greens64, tmp_path, monkeypatch, seed_chunk):
    """gt_monte_carlo (capi.cpp:345-369) against the reference library, seed for seed. The
    seeds stream through in chunks (GT_MC_SEED_CHUNK=4 forces two chunks of 6 seeds)."""
    if seed_chunk:
        monkeypatch.setenv("GT_MC_SEED_CHUNK", seed_chunk)
    gdir = tmp_path / "g"
    oracle.save_greens_dir(greens64, gdir)
    var = _write(tmp_path / "var.txt", "beta 0.017\nseed 7\n")
    from paper_2307_12119_b200 import inputs
    import dataclasses
    p = inputs.power_map(dataclasses.replace(inputs.CONFIGS["cfg0"], n=64), 3) * 0.3
    seeds = (C.c_ulonglong * 6)(1, 2, 3, 5, 8, 13)
    out = []
    for L in (b200lib, oracle.ref_lib()):
        g = C.c_void_p()
        assert L.gt_greens_load(str(gdir).encode(), C.byref(g)) == 0
        f = C.c_void_p()
        assert L.gt_field_create(64, greens64.pitch, b"watts", C.byref(f)) == 0
        np.ctypeslib.as_array(L.gt_field_data(f), shape=(64, 64))[...] = p
        csv_path = tmp_path / f"mc_{len(out)}.csv"
        mean, sd = C.c_double(), C.c_double()
        st = L.gt_monte_carlo(g, var, None, 20.0, f, seeds, 6, 4, str(csv_path).encode(), C.byref(mean), C.byref(sd))
        assert st == 0, L.gt_last_error()
        rows = list(csv.DictReader(open(csv_path)))
        out.append((mean.value, sd.value, [(int(r["seed"]), float(r["max_rise"]), float(r["mean_rise"])) for r in rows]))
    (mb, sb, rb), (mr, sr, rr) = out
    print(f"mean_max {mb:.9f} vs {mr:.9f}; std {sb:.3e} vs {sr:.3e}")
    assert mb == pytest.approx(mr, rel=1e-9, abs=1e-9)
    assert sb == pytest.approx(sr, rel=1e-6, abs=1e-9)
    for a, b in zip(rb, rr):
        assert a[0] == b[0]
        assert a[1] == pytest.approx(b[1], rel=1e-10)
        assert a[2] == pytest.approx(b[2], rel=1e-10)
