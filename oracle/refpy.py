"""oracle/refpy.py — TEST INFRASTRUCTURE ONLY.

ctypes access to the CPU oracle built by ``oracle/Makefile``:
  * ``ref_lib()``     — the UNCHANGED reference library (49 gt_* symbols) compiled
                        from /root/reference/proj against the FFTW/Eigen subset shims;
  * ``restate_lib()`` — batch drivers over the same reference core (mode A) and
                        the fp64 restatement of the north-star fixed point (mode B).
Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU legs import this
module; the product never does. Parity status: pinned to the reference's own
code for mode A (the arithmetic IS the reference source); FFTW and Eigen are
replaced by shims validated against numpy (tests/test_oracle.py) — the
reference pins neither library version (CMakeLists.txt:12-18), so that
boundary is "parity unpinned" beyond the DFT definition itself.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REF_SO = HERE / "_ref" / "libgreentherm_ref.so"
RESTATE_SO = HERE / "_ref" / "libgt_restate.so"

dbl, cint, vp = C.c_double, C.c_int, C.c_void_p
pdbl = C.POINTER(C.c_double)
pint = C.POINTER(C.c_int)


class RefGreens(C.Structure):
    _fields_ = [("n", cint), ("pitch", dbl), ("phi", dbl), ("kappa_inf", dbl), ("alpha", dbl), ("beta", dbl),
                ("mu", dbl), ("capacitance", dbl), ("rand_scale", dbl), ("f_sp0", pdbl), ("g_sp0", pdbl),
                ("f_det", pdbl), ("f_rand", pdbl), ("p_var", pdbl)]


def available() -> bool:
    return REF_SO.exists() and RESTATE_SO.exists()


def build_if_possible() -> bool:
    """Build the oracle when the reference sources are present (this container)."""
    if available():
        return True
    if not Path("/root/reference/proj").exists():
        return False
    import subprocess
    subprocess.run(["make", "-C", str(HERE), "-j8"], check=True, capture_output=True)
    return available()


_REF = None
_RST = None


def ref_lib() -> C.CDLL:
    global _REF
    if _REF is None:
        from paper_2307_12119_b200.api import bind
        _REF = bind(C.CDLL(str(REF_SO)), extension=False)
    return _REF


def restate_lib() -> C.CDLL:
    global _RST
    if _RST is None:
        L = C.CDLL(str(RESTATE_SO))
        L.ref_mc_batch.restype = dbl
        L.ref_mc_batch.argtypes = [C.POINTER(RefGreens), pdbl, pdbl, cint, dbl, cint, dbl, cint, cint, pdbl, pdbl,
                                   pdbl, pint]
        L.ref_greens_save_dir.restype = cint
        L.ref_greens_save_dir.argtypes = [C.POINTER(RefGreens), C.c_char_p]
        L.ref_impulse_response.restype = cint
        L.ref_impulse_response.argtypes = [cint, dbl, dbl, pdbl]
        L.ref_calibrate.restype = cint
        L.ref_calibrate.argtypes = [cint, dbl, dbl, dbl, dbl, cint, cint, C.POINTER(RefGreens)]
        L.ref_fixed_point_batch.restype = dbl
        L.ref_fixed_point_batch.argtypes = [C.POINTER(RefGreens), pdbl, pdbl, cint, dbl, dbl, cint, cint, dbl, dbl,
                                            dbl, cint, cint, pdbl, pint, pint]
        L.ref_fixed_point_rand_batch.argtypes = [C.POINTER(RefGreens), pdbl, pdbl, cint, dbl, dbl, cint, cint, dbl, dbl,
                                            dbl, cint, cint, pdbl, pint, pint]
        L.ref_fixed_point_rand_batch.restype = dbl
        L.ref_trace_leak_batch.restype = dbl
        L.ref_trace_leak_batch.argtypes = [C.POINTER(RefGreens), C.POINTER(C.c_int), C.c_longlong, pdbl, cint, pdbl,
                                           C.c_longlong, cint, dbl, cint, cint, cint, dbl, cint, cint, pdbl, pint]
        _RST = L
    return _RST


def _p(a):
    return None if a is None else a.ctypes.data_as(pdbl)


class _Keep:
    """RefGreens plus the arrays it points into (kept alive together)."""

    def __init__(self, g):
        self.arrs = {k: (None if getattr(g, k, None) is None else np.ascontiguousarray(getattr(g, k), np.float64))
                     for k in ("f_sp0", "g_sp0", "f_det", "f_rand", "p_var")}
        self.s = RefGreens(g.n, g.pitch, g.phi, g.kappa_inf, g.alpha, g.beta, g.mu, g.capacitance, g.rand_scale,
                           *(_p(self.arrs[k]) for k in ("f_sp0", "g_sp0", "f_det", "f_rand", "p_var")))


def mc_batch(g, p_dyn, var, leak_frac=0.3, mu_per_sample=1, with_rand=1, jobs=None, beta_l=-10.0, want_maps=True):
    """Reference run_one per pair (mode A). Returns (maps, max, mean, status, seconds)."""
    k = _Keep(g)
    p = np.ascontiguousarray(p_dyn, np.float64)
    v = np.ascontiguousarray(var, np.float64)
    B = p.shape[0]
    out = np.empty_like(p) if want_maps else None
    mx, mean, st = np.empty(B), np.empty(B), np.empty(B, np.int32)
    secs = restate_lib().ref_mc_batch(C.byref(k.s), _p(p), _p(v), B, leak_frac, mu_per_sample, beta_l, with_rand,
                                      jobs or os.cpu_count() or 1, _p(out), _p(mx), _p(mean),
                                      st.ctypes.data_as(pint))
    return out, mx, mean, st, secs


def fixed_point_batch(g, p_dyn, var, leak_frac=0.3, beta=0.017, law=1, kirchhoff=0, t_ambient=318.15, eta=1.3,
                      tol=1e-4, max_iters=50, jobs=None, with_rand=0):
    """Mode B restatement (with_rand: + the reference's shift-variant term each iteration,
    restate.h ref_fixed_point_rand_batch). Returns (maps, iters, status, seconds)."""
    k = _Keep(g)
    p = np.ascontiguousarray(p_dyn, np.float64)
    v = np.ascontiguousarray(var, np.float64)
    B = p.shape[0]
    out = np.empty_like(p)
    it, st = np.empty(B, np.int32), np.empty(B, np.int32)
    fn = restate_lib().ref_fixed_point_rand_batch if with_rand else restate_lib().ref_fixed_point_batch
    secs = fn(C.byref(k.s), _p(p), _p(v), B, leak_frac, beta, law, kirchhoff,
                                               t_ambient, eta, tol, max_iters, jobs or os.cpu_count() or 1, _p(out),
                                               it.ctypes.data_as(pint), st.ctypes.data_as(pint))
    return out, it, st, secs


def trace_leak_batch(g, blk, sched, leak0, dt, window, law=0, beta=0.017, out_stride=1, jobs=None):
    """Config-3 oracle: blk [B|1, n, n] int, sched [B, steps, nblk], leak0 [B|1, n, n].
    Returns (frames [B, steps // out_stride, n, n], status, seconds)."""
    k = _Keep(g)
    blk = np.ascontiguousarray(blk, np.int32)
    sched = np.ascontiguousarray(sched, np.float64)
    leak0 = np.ascontiguousarray(leak0, np.float64)
    B, steps, nblk = sched.shape
    n = g.n
    nn = n * n
    out = np.zeros((B, steps // out_stride, n, n))
    st = np.empty(B, np.int32)
    secs = restate_lib().ref_trace_leak_batch(
        C.byref(k.s), blk.ctypes.data_as(C.POINTER(C.c_int)), nn if blk.shape[0] > 1 else 0, _p(sched), nblk,
        _p(leak0), nn if leak0.shape[0] > 1 else 0, B, dt, steps, window, law, beta, out_stride,
        jobs or os.cpu_count() or 1, _p(out), st.ctypes.data_as(pint))
    return out, st, secs


def save_greens_dir(g, path) -> None:
    k = _Keep(g)
    rc = restate_lib().ref_greens_save_dir(C.byref(k.s), str(path).encode())
    if rc:
        raise RuntimeError(f"ref_greens_save_dir failed ({rc})")


def impulse_response(n, die_edge=0.016, k_die=130.0) -> np.ndarray:
    out = np.empty((n, n))
    rc = restate_lib().ref_impulse_response(n, die_edge, k_die, _p(out))
    if rc:
        raise RuntimeError(f"ref_impulse_response failed ({rc})")
    return out


def calibrate(n, die_edge=0.016, beta=0.017, dopant_spread=0.0, leak_total=15.0, fit_rand_scale=True,
              fit_transient=False) -> dict:
    """The reference calibrate() -> dict of GreensSet arrays/scalars."""
    bufs = {k: np.zeros((n, n)) for k in ("f_sp0", "g_sp0", "f_det", "f_rand", "p_var")}
    s = RefGreens(n, 0, 0, 0, 0, 0, 0, 0, 0, *(_p(bufs[k]) for k in ("f_sp0", "g_sp0", "f_det", "f_rand", "p_var")))
    rc = restate_lib().ref_calibrate(n, die_edge, beta, dopant_spread, leak_total, int(fit_rand_scale),
                                     int(fit_transient), C.byref(s))
    if rc:
        raise RuntimeError(f"reference calibrate failed (status class {rc})")
    out = dict(bufs)
    for k in ("n", "pitch", "phi", "kappa_inf", "alpha", "beta", "mu", "capacitance", "rand_scale"):
        out[k] = getattr(s, k)
    return out
