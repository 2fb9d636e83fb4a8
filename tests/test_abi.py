"""The C-ABI boundary (CPU only: no compute calls need a GPU here).

Checks that libgreentherm_b200.so loads, exports every function include/*.h
declares, that the host-side handle API behaves like the reference's
(same status codes, thread-local error text, file formats the reference
reads back), and that a solve without a CUDA device fails loudly instead of
falling back to the CPU.
"""
import ctypes as C
import re
from pathlib import Path

import numpy as np
import pytest

from conftest import ROOT, has_gpu

HEADERS = sorted((ROOT / "include").glob("*.h"))


def declared_functions():
    names = set()
    for h in HEADERS:
        txt = re.sub(r"/\*.*?\*/", "", h.read_text(), flags=re.S)
        for m in re.finditer(r"\b(gt_[a-z0-9_]+)\s*\(", txt):
            names.add(m.group(1))
    return sorted(names)


def test_headers_declare_reference_surface():
    from paper_2307_12119_b200.api import CORE_SYMBOLS
    names = declared_functions()
    assert set(CORE_SYMBOLS) <= set(names)
    assert len(CORE_SYMBOLS) == 49  # reference greentherm.h exports 49 entry points


def test_library_exports_every_declared_symbol(b200lib):
    lib = C.CDLL(str(Path(b200lib._name)))
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing


def test_status_names(b200lib):
    assert b200lib.gt_status_name(0) == b"ok"
    assert b200lib.gt_status_name(3) == b"solver"
    assert b200lib.gt_status_name(5) == b"internal"


def test_field_roundtrip_and_compensated_sum(b200lib, tmp_path):
    L = b200lib
    f = C.c_void_p()
    assert L.gt_field_create(8, 0.5, b"watts", C.byref(f)) == 0
    vals = np.array([1e16, 1.0, -1e16, 1.0] + [0.0] * 60)
    for k, v in enumerate(vals):
        L.gt_field_set(f, k // 8, k % 8, v)
    assert L.gt_field_sum(f) == 2.0  # Neumaier (reference field.cpp:45-57); naive gives 1.0
    p = tmp_path / "f.map"
    assert L.gt_field_save(f, str(p).encode()) == 0
    g = C.c_void_p()
    assert L.gt_field_load(str(p).encode(), C.byref(g)) == 0
    assert L.gt_field_n(g) == 8 and L.gt_field_pitch(g) == 0.5 and L.gt_field_unit(g) == b"watts"
    data = np.ctypeslib.as_array(L.gt_field_data(g), shape=(64,))
    np.testing.assert_array_equal(data, vals)
    L.gt_field_free(f)
    L.gt_field_free(g)


def test_config_errors_are_thread_local_and_classed(b200lib, tmp_path):
    L = b200lib
    f = C.c_void_p()
    assert L.gt_field_create(1, 0.5, b"watts", C.byref(f)) == 2
    assert L.gt_last_error_stage() == b"field"
    assert L.gt_field_create(4, 0.5, b"furlongs", C.byref(f)) == 2
    assert b"unknown field unit" in L.gt_last_error()
    assert L.gt_field_load(str(tmp_path / "missing.map").encode(), C.byref(f)) == 2


def test_reference_written_greens_dir_loads(b200lib, oracle, greens64, tmp_path):
    """Our loader reads a GreensSet directory written by the reference's save_greens."""
    d = tmp_path / "gs"
    oracle.save_greens_dir(greens64, d)
    L = b200lib
    g = C.c_void_p()
    assert L.gt_greens_load(str(d).encode(), C.byref(g)) == 0, L.gt_last_error()
    assert L.gt_greens_n(g) == 64
    assert L.gt_greens_alpha(g) == greens64.alpha
    assert L.gt_greens_mu(g) == greens64.mu
    f = C.c_void_p()
    assert L.gt_greens_field(g, b"f_sp0", C.byref(f)) == 0
    np.testing.assert_array_equal(np.ctypeslib.as_array(L.gt_field_data(f), shape=(64, 64)), greens64.f_sp0)
    assert L.gt_greens_field(g, b"nope", C.byref(f)) == 2
    # and the reference reads what we write
    d2 = tmp_path / "gs2"
    assert L.gt_greens_save(g, str(d2).encode()) == 0
    R = oracle.ref_lib()
    rg = C.c_void_p()
    assert R.gt_greens_load(str(d2).encode(), C.byref(rg)) == 0, R.gt_last_error()
    assert R.gt_greens_alpha(rg) == greens64.alpha
    R.gt_greens_free(rg)
    L.gt_greens_free(g)


def test_greens_from_arrays_validates(b200lib, greens64):
    bad = np.array(greens64.f_sp0)
    bad[0, 0] = bad.max() * 2  # peak away from the source cell (greens.cpp:99-103)
    import dataclasses
    g = dataclasses.replace(greens64, f_sp0=bad, g_sp0=None)
    with pytest.raises(Exception) as e:
        g.to_handle(b200lib)
    assert "peak" in str(e.value)


def test_error_metrics(b200lib):
    L = b200lib
    a, b = C.c_void_p(), C.c_void_p()
    L.gt_field_create(4, 1.0, b"kelvin", C.byref(a))
    L.gt_field_create(4, 1.0, b"kelvin", C.byref(b))
    L.gt_field_set(a, 1, 1, 3.0)
    L.gt_field_set(b, 1, 2, 4.0)

    class Rep(C.Structure):
        _fields_ = [("mae", C.c_double), ("max_err", C.c_double), ("pct", C.c_double), ("maxpct", C.c_double),
                    ("hit", C.c_int)]
    r = Rep()
    assert L.gt_error_metrics(a, b, C.byref(r)) == 0
    assert r.mae == pytest.approx(7.0 / 16) and r.max_err == 4.0 and r.hit == 1
    assert r.pct == pytest.approx(100 * 7.0 / 16 / 4.0)


@pytest.mark.skipif(has_gpu(), reason="checks the no-device failure path")
def test_solve_without_device_fails_loudly(b200lib, greens64):
    from paper_2307_12119_b200.api import DeviceGreens, GtError
    with pytest.raises(GtError) as e:
        DeviceGreens(greens64)
    assert e.value.status == 5 and e.value.stage == "device"
    assert b200lib.gt_device_count() == 0


def test_field_binary_sidecar(b200lib, tmp_path):
    """gt_field_save writes the reference text format plus a binary sidecar; loads prefer
    a fresh sidecar and fall back to the text when the text no longer matches it."""
    import ctypes as C
    import numpy as np
    L = b200lib
    n = 8
    f = C.c_void_p()
    assert L.gt_field_create(n, 0.001, b"kelvin", C.byref(f)) == 0
    vals = np.ctypeslib.as_array(L.gt_field_data(f), shape=(n, n))
    vals[...] = np.arange(n * n).reshape(n, n) * 0.1 + 1e-3
    path = tmp_path / "t.map"
    assert L.gt_field_save(f, str(path).encode()) == 0
    assert (tmp_path / "t.map.bin").exists()
    g = C.c_void_p()
    assert L.gt_field_load(str(path).encode(), C.byref(g)) == 0
    np.testing.assert_array_equal(np.ctypeslib.as_array(L.gt_field_data(g), shape=(n, n)), vals)
    L.gt_field_free(g)
    # edit the text (another tool): the stale sidecar must be ignored
    lines = path.read_text().splitlines()
    lines[1] = " ".join(["5"] * n)
    path.write_text("\n".join(lines) + "\n")
    assert L.gt_field_load(str(path).encode(), C.byref(g)) == 0
    got = np.ctypeslib.as_array(L.gt_field_data(g), shape=(n, n))
    assert (got[0] == 5).all()
    L.gt_field_free(g)
    L.gt_field_free(f)


def test_field_sidecar_same_size_rewrite_with_copied_mtime(b200lib, tmp_path):
    """A text rewritten to the SAME byte size whose mtime is then set back (cp -p / rsync /
    tar keep mtimes) must not be served from the stale sidecar: the sidecar records a
    content fingerprint of the text, not only its size and age."""
    import ctypes as C
    import os
    import numpy as np
    L = b200lib
    n = 8
    f = C.c_void_p()
    assert L.gt_field_create(n, 0.001, b"kelvin", C.byref(f)) == 0
    vals = np.ctypeslib.as_array(L.gt_field_data(f), shape=(n, n))
    vals[...] = 1.25
    path = tmp_path / "t.map"
    assert L.gt_field_save(f, str(path).encode()) == 0
    st = os.stat(path)
    text = path.read_text()
    edited = text.replace("1.25", "2.25", 3)  # same length, different values
    assert len(edited) == len(text) and edited != text
    path.write_text(edited)
    os.utime(path, ns=(st.st_atime_ns, st.st_mtime_ns - 10**9))  # older than the sidecar
    g = C.c_void_p()
    assert L.gt_field_load(str(path).encode(), C.byref(g)) == 0
    got = np.ctypeslib.as_array(L.gt_field_data(g), shape=(n, n))
    assert (got == 2.25).sum() == 3
    L.gt_field_free(g)
    L.gt_field_free(f)


def test_error_metrics_match_reference_library(b200lib, oracle):
    """gt_error_metrics (reference capi.cpp:333 -> error_metrics, solver.cpp:289-336) on
    random fields against the reference library itself: MAE, max error, % of the
    reference's max rise, and the hotspot hit (Chebyshev distance <= 1)."""
    import numpy as np
    rng = np.random.default_rng(11)

    class Rep(C.Structure):
        _fields_ = [("mae", C.c_double), ("max_err", C.c_double), ("pct", C.c_double), ("maxpct", C.c_double),
                    ("hit", C.c_int)]
    for trial in range(6):
        n = int(rng.choice([4, 16, 64]))
        a_v = rng.uniform(0, 50, (n, n))
        b_v = a_v + rng.normal(0, 2.0, (n, n))
        if trial % 2:
            b_v[rng.integers(n), rng.integers(n)] += 100.0  # move the reference hotspot
        reps = []
        for L in (b200lib, oracle.ref_lib()):
            a, b = C.c_void_p(), C.c_void_p()
            assert L.gt_field_create(n, 0.001, b"kelvin", C.byref(a)) == 0
            assert L.gt_field_create(n, 0.001, b"kelvin", C.byref(b)) == 0
            np.ctypeslib.as_array(L.gt_field_data(a), shape=(n, n))[...] = a_v
            np.ctypeslib.as_array(L.gt_field_data(b), shape=(n, n))[...] = b_v
            r = Rep()
            assert L.gt_error_metrics(a, b, C.byref(r)) == 0
            reps.append((r.mae, r.max_err, r.pct, r.maxpct, r.hit))
            L.gt_field_free(a)
            L.gt_field_free(b)
        ours, ref = reps
        assert ours[4] == ref[4]
        np.testing.assert_allclose(ours[:4], ref[:4], rtol=1e-12, atol=0)
