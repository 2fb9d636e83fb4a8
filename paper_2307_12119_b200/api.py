"""ctypes mirror of include/greentherm.h and include/greentherm_b200.h.

:func:`bind` declares the prototypes of the 49 reference entry points on any
CDLL exporting them — this library, or the reference library compiled by
``oracle/Makefile`` — so parity tests drive both through the identical ABI.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_LIBNAME = "libgreentherm_b200.so"

GT_FP32, GT_FP64 = 0, 1
# per-sample status bits (include/greentherm_b200.h GT_SAMPLE_*; gt_device.h GTD_ST_*)
(GT_SAMPLE_BAD_POWER, GT_SAMPLE_BAD_VAR, GT_SAMPLE_RUNAWAY_DET, GT_SAMPLE_RUNAWAY_RAND, GT_SAMPLE_NONFINITE,
 GT_SAMPLE_NOCONVERGE, GT_SAMPLE_KIRCHHOFF, GT_SAMPLE_ILLCOND) = 1, 2, 4, 8, 16, 32, 64, 128

vp = C.c_void_p
pvp = C.POINTER(C.c_void_p)
dbl = C.c_double
pdbl = C.POINTER(C.c_double)
cint = C.c_int
cstr = C.c_char_p

# (name, restype, argtypes) — reference greentherm.h
_CORE = [
    ("gt_status_name", cstr, [cint]),
    ("gt_last_error", cstr, []),
    ("gt_last_error_stage", cstr, []),
    ("gt_field_create", cint, [cint, dbl, cstr, pvp]),
    ("gt_field_load", cint, [cstr, pvp]),
    ("gt_field_save", cint, [vp, cstr]),
    ("gt_field_free", None, [vp]),
    ("gt_field_n", cint, [vp]),
    ("gt_field_pitch", dbl, [vp]),
    ("gt_field_unit", cstr, [vp]),
    ("gt_field_get", dbl, [vp, cint, cint]),
    ("gt_field_set", None, [vp, cint, cint, dbl]),
    ("gt_field_data", pdbl, [vp]),
    ("gt_field_max", dbl, [vp]),
    ("gt_field_sum", dbl, [vp]),
    ("gt_field_render", cint, [vp, cstr, cint]),
    ("gt_write_default_stack", cint, [cstr]),
    ("gt_write_default_variation", cint, [cstr]),
    ("gt_calibrate", cint, [cstr, cstr, vp, dbl, pvp, pdbl]),
    ("gt_greens_save", cint, [vp, cstr]),
    ("gt_greens_load", cint, [cstr, pvp]),
    ("gt_greens_free", None, [vp]),
    ("gt_greens_n", cint, [vp]),
    ("gt_greens_alpha", dbl, [vp]),
    ("gt_greens_beta", dbl, [vp]),
    ("gt_greens_mu", dbl, [vp]),
    ("gt_greens_capacitance", dbl, [vp]),
    ("gt_greens_kappa_inf", dbl, [vp]),
    ("gt_greens_field", cint, [vp, cstr, pvp]),
    ("gt_result_count", cint, [vp]),
    ("gt_result_time", dbl, [vp, cint]),
    ("gt_result_map", cint, [vp, cint, pvp]),
    ("gt_result_free", None, [vp]),
    ("gt_solve_steady", cint, [vp, vp, cint, pvp, pdbl]),
    ("gt_solve_step", cint, [vp, vp, pdbl, cint, cint, pvp, pdbl]),
    ("gt_trace_load", cint, [cstr, pvp]),
    ("gt_trace_create", cint, [dbl, pvp]),
    ("gt_trace_push", cint, [vp, vp]),
    ("gt_trace_save", cint, [vp, cstr]),
    ("gt_trace_frames", cint, [vp]),
    ("gt_trace_dt", dbl, [vp]),
    ("gt_trace_free", None, [vp]),
    ("gt_solve_trace", cint, [vp, vp, cint, cint, pvp, pdbl]),
    ("gt_oracle_steady", cint, [cstr, cstr, vp, vp, cint, cint, pvp, C.POINTER(cint)]),
    ("gt_oracle_transient", cint, [cstr, cstr, vp, vp, cint, pdbl, cint, dbl, pvp]),
    ("gt_error_metrics", cint, [vp, vp, vp]),
    ("gt_monte_carlo", cint, [vp, cstr, vp, dbl, vp, C.POINTER(C.c_ulonglong), cint, cint, cstr, pdbl, pdbl]),
    ("gt_write_builtin_suite", cint, [cstr, cstr]),
    ("gt_validate_suite", cint, [cstr, cstr, cint, C.POINTER(cint), C.POINTER(cint)]),
]
CORE_SYMBOLS = [n for n, _, _ in _CORE]


class BatchOpts(C.Structure):
    _fields_ = [("leak_frac", dbl), ("mu_per_sample", cint), ("with_rand", cint), ("chunk", cint),
                ("exponent_cap", dbl), ("fp64_check", dbl)]


class SampleStats(C.Structure):
    _fields_ = [("sum_leak", dbl), ("sum_applied", dbl), ("sum_rise", dbl), ("max_rise", dbl),
                ("mean_rise", dbl), ("mu", dbl), ("max_bits", C.c_ulonglong), ("status", cint),
                ("max_rden2", C.c_float)]


class FPOpts(C.Structure):
    _fields_ = [("leak_frac", dbl), ("law", cint), ("kirchhoff", cint), ("beta", dbl), ("t_ambient", dbl),
                ("eta", dbl), ("tol", dbl), ("max_iters", cint), ("chunk", cint), ("fp32_stage_tol", dbl),
                ("with_rand", cint), ("accel", cint), ("warm_start", cint)]


SAMPLE_STATS_DTYPE = np.dtype([("sum_leak", "f8"), ("sum_applied", "f8"), ("sum_rise", "f8"),
                               ("max_rise", "f8"), ("mean_rise", "f8"), ("mu", "f8"),
                               ("max_bits", "u8"), ("status", "i4"), ("max_rden2", "f4")])

# greentherm_b200.h
class TraceOpts(C.Structure):
    _fields_ = [("dt", dbl), ("steps", cint), ("window", cint), ("law", cint), ("beta", dbl),
                ("out_stride", cint), ("chunk", cint)]


_EXT = [
    ("gt_greens_from_arrays", cint, [cint, dbl, pdbl, pdbl, dbl, dbl, dbl, dbl, dbl, dbl, dbl, pdbl, pdbl,
                                     pdbl, pvp]),
    ("gt_greens_to_device", cint, [vp, cint, cint, pvp]),
    ("gt_device_greens_free", None, [vp]),
    ("gt_device_greens_precision", cint, [vp]),
    ("gt_batch_opts_default", None, [C.POINTER(BatchOpts)]),
    ("gt_mc_batch", cint, [vp, vp, vp, cint, C.POINTER(BatchOpts), vp, pdbl, pdbl, C.POINTER(cint), pdbl]),
    ("gt_mc_batch_device", cint, [vp, vp, vp, cint, C.POINTER(BatchOpts), vp, vp, vp]),
    ("gt_mc_scratch_bytes", C.c_size_t, [cint, cint]),
    ("gt_mc_kernel_launches", cint, [cint, cint]),
    ("gt_device_count", cint, []),
    ("gt_fp_opts_default", None, [C.POINTER(FPOpts)]),
    ("gt_fp_batch", cint, [vp, vp, vp, cint, C.POINTER(FPOpts), vp, C.POINTER(cint), C.POINTER(cint), pdbl, pdbl]),
    ("gt_fp_batch_device", cint, [vp, vp, vp, cint, C.POINTER(FPOpts), vp, vp, vp, vp, vp, vp]),
    ("gt_fp_scratch_bytes", C.c_size_t, [cint, cint]),
    ("gt_trace_opts_default", None, [C.POINTER(TraceOpts)]),
    ("gt_trace_batch_device", cint, [vp, vp, C.c_longlong, vp, cint, vp, C.c_longlong, cint, C.POINTER(TraceOpts),
                                     vp, vp, vp]),
    ("gt_trace_scratch_bytes", C.c_size_t, [cint, cint, cint]),
    ("gt_modal_kernel", cint, [cstr, C.POINTER(cint), pdbl]),
    ("gt_var_model", cint, [vp, dbl, dbl]),
    ("gt_var_generate_device", cint, [vp, vp, cint, vp, vp]),
    ("gt_mc_batch_seeded", cint, [vp, vp, vp, cint, C.POINTER(BatchOpts), vp, pdbl, pdbl, C.POINTER(cint), pdbl]),
    ("gt_large_geometry", cint, [vp, C.POINTER(cint), C.POINTER(cint)]),
    ("gt_large_rows_fwd", cint, [vp, vp, cint, vp, vp, vp]),
    ("gt_large_row_layout", cint, [vp, C.POINTER(cint)]),
    ("gt_large_lowmode_state_bytes", C.c_size_t, []),
    ("gt_large_lowmode_partial_blocks", cint, [cint]),
    ("gt_large_lowmode_init", cint, [vp, vp]),
    ("gt_large_lowmode_project", cint, [vp, vp, cint, cint, cint, vp, vp, vp]),
    ("gt_large_lowmode_mix", cint, [vp, vp, cint, C.c_double, vp, vp]),
    ("gt_large_lowmode_apply", cint, [vp, vp, cint, cint, cint, vp, vp]),
    ("gt_large_cols", cint, [vp, vp, cint, cint, cint, vp, vp, vp, vp]),
    ("gt_large_rows_inv", cint, [vp, vp, cint, cint, vp, vp, vp, vp, vp, C.POINTER(FPOpts), vp, vp, vp]),
    ("gt_large_cols_peer", cint, [vp, vp, cint, cint, cint, cint, vp, vp, vp, cint, vp]),
    ("gt_ipc_alloc", cint, [C.c_size_t, C.POINTER(vp), vp]),
    ("gt_ipc_open", cint, [vp, C.POINTER(vp)]),
    ("gt_ipc_close", cint, [vp]),
    ("gt_ipc_free", cint, [vp]),
    ("gt_large_rows_inv_accel", cint, [vp, vp, cint, cint, vp, vp, vp, vp, vp, C.POINTER(FPOpts), vp, vp, vp, vp,
                                       C.c_double, C.c_double, vp]),
    ("gt_profile_begin", cint, [vp]),
    ("gt_profile_begin_mode", cint, [vp, cint]),
    ("gt_profile_end", cint, [vp, pdbl, C.POINTER(C.c_longlong), C.POINTER(C.c_longlong)]),
    ("gt_kernel_launches", C.c_longlong, [vp]),
]
EXT_SYMBOLS = [n for n, _, _ in _EXT]


def bind(cdll: C.CDLL, extension: bool = True) -> C.CDLL:
    """Declare prototypes on ``cdll`` (the reference library has no extension)."""
    for name, res, args in _CORE + (_EXT if extension else []):
        fn = getattr(cdll, name)
        fn.restype = res
        fn.argtypes = args
    return cdll


def library_path() -> Path:
    # GT_B200_LIB selects an in-tree tuning variant built by ``build.py --variant``.
    import os
    alt = os.environ.get("GT_B200_LIB")
    return Path(alt) if alt else _HERE / _LIBNAME


_LIB: C.CDLL | None = None


def lib() -> C.CDLL:
    """Load the B200 library (fails loudly if it has not been built)."""
    global _LIB
    if _LIB is None:
        p = library_path()
        if not p.exists():
            raise RuntimeError(f"{p} is missing: run `python -m paper_2307_12119_b200.build` (no CPU fallback)")
        _LIB = bind(C.CDLL(str(p)))
    return _LIB


class GtError(RuntimeError):
    def __init__(self, status: int, stage: str, msg: str):
        super().__init__(f"status={status} stage={stage} msg={msg}")
        self.status, self.stage, self.msg = status, stage, msg


def check(cdll: C.CDLL, status: int) -> None:
    if status != 0:
        raise GtError(status, cdll.gt_last_error_stage().decode(), cdll.gt_last_error().decode())


def _p(a: np.ndarray | None):
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(pdbl)


@dataclass
class GreensArrays:
    """A GreensSet as plain arrays (reference greens.hpp:18-39)."""
    n: int
    pitch: float
    f_sp0: np.ndarray
    g_sp0: np.ndarray
    phi: float
    kappa_inf: float
    alpha: float
    beta: float
    mu: float
    capacitance: float = 0.0
    rand_scale: float = 1.0
    f_det: np.ndarray | None = None
    f_rand: np.ndarray | None = None
    p_var: np.ndarray | None = None

    def to_handle(self, cdll: C.CDLL | None = None) -> C.c_void_p:
        cdll = cdll or lib()
        h = C.c_void_p()
        arrs = [None if a is None else np.ascontiguousarray(a, dtype=np.float64)
                for a in (self.f_sp0, self.g_sp0, self.f_det, self.f_rand, self.p_var)]
        check(cdll, cdll.gt_greens_from_arrays(self.n, self.pitch, _p(arrs[0]), _p(arrs[1]), self.phi,
                                               self.kappa_inf, self.alpha, self.beta, self.mu,
                                               self.capacitance, self.rand_scale, _p(arrs[2]), _p(arrs[3]),
                                               _p(arrs[4]), C.byref(h)))
        return h

    @staticmethod
    def from_npz(path) -> "GreensArrays":
        z = np.load(path)
        g = lambda k, d=None: (z[k] if k in z.files else d)  # noqa: E731
        return GreensArrays(n=int(z["n"]), pitch=float(z["pitch"]), f_sp0=z["f_sp0"], g_sp0=z["g_sp0"],
                            phi=float(z["phi"]), kappa_inf=float(z["kappa_inf"]), alpha=float(z["alpha"]),
                            beta=float(z["beta"]), mu=float(z["mu"]),
                            capacitance=float(g("capacitance", 0.0)), rand_scale=float(g("rand_scale", 1.0)),
                            f_det=g("f_det"), f_rand=g("f_rand"), p_var=g("p_var"))


class DeviceGreens:
    """Prepared device-resident GreensSet (gt_greens_to_device)."""

    def __init__(self, greens: GreensArrays, precision: int = GT_FP32, device: int = 0):
        L = lib()
        self.n = greens.n
        self.precision = precision
        self._g = greens.to_handle(L)
        self._d = C.c_void_p()
        try:
            check(L, L.gt_greens_to_device(self._g, precision, device, C.byref(self._d)))
        except Exception:
            L.gt_greens_free(self._g)
            self._g = C.c_void_p()
            raise

    @property
    def handle(self):
        return self._d

    def close(self):
        L = lib()
        if self._d:
            L.gt_device_greens_free(self._d)
            self._d = C.c_void_p()
        if self._g:
            L.gt_greens_free(self._g)
            self._g = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def opts(self, leak_frac=0.3, mu_per_sample=1, with_rand=1, chunk=0, exponent_cap=6.0,
             fp64_check=0.0) -> BatchOpts:
        """fp64_check: conditioning threshold of the fp64 re-solve (0 = default 1e4, < 0 = off)."""
        return BatchOpts(leak_frac, mu_per_sample, with_rand, chunk, exponent_cap, fp64_check)

    def mc_batch_host(self, p_dyn: np.ndarray, var: np.ndarray, opts: BatchOpts | None = None,
                      want_maps: bool = True):
        """End-to-end batch from host arrays; returns (maps|None, max, mean, status, ms)."""
        L = lib()
        dt = np.float64 if self.precision == GT_FP64 else np.float32
        p = np.ascontiguousarray(p_dyn, dtype=dt)
        v = np.ascontiguousarray(var, dtype=dt)
        B = p.shape[0]
        out = np.empty_like(p) if want_maps else None
        mx, mean = np.empty(B), np.empty(B)
        st = np.empty(B, dtype=np.int32)
        ms = C.c_double()
        o = opts or self.opts()
        check(L, L.gt_mc_batch(self._d, p.ctypes.data_as(vp), v.ctypes.data_as(vp), B, C.byref(o),
                               None if out is None else out.ctypes.data_as(vp), mx.ctypes.data_as(pdbl),
                               mean.ctypes.data_as(pdbl), st.ctypes.data_as(C.POINTER(cint)), C.byref(ms)))
        return out, mx, mean, st, ms.value

    def var_model(self, sigma_over_mu: float = 0.10, range_frac: float = 0.5) -> None:
        """Prepare the seeded device variation model (include/greentherm_b200.h gt_var_model)."""
        check(lib(), lib().gt_var_model(self._d, sigma_over_mu, range_frac))

    def var_generate_device(self, seeds_ptr: int, batch: int, out_ptr: int, stream: int | None = None) -> None:
        sp = None if stream is None else C.c_void_p(stream if stream else 1)
        check(lib(), lib().gt_var_generate_device(self._d, C.c_void_p(seeds_ptr), batch, C.c_void_p(out_ptr), sp))

    def mc_batch_seeded_host(self, p_dyn: np.ndarray, seeds: np.ndarray, opts: BatchOpts | None = None,
                             want_maps: bool = True):
        """Host power maps + host seeds (variation generated on the device);
        returns (maps|None, max, mean, status, ms)."""
        L = lib()
        dt = np.float64 if self.precision == GT_FP64 else np.float32
        p = np.ascontiguousarray(p_dyn, dtype=dt)
        sd = np.ascontiguousarray(seeds, dtype=np.uint64)
        B = p.shape[0]
        out = np.empty_like(p) if want_maps else None
        mx, mean = np.empty(B), np.empty(B)
        st = np.empty(B, dtype=np.int32)
        ms = C.c_double()
        o = opts or self.opts()
        check(L, L.gt_mc_batch_seeded(self._d, p.ctypes.data_as(vp), sd.ctypes.data_as(vp), B, C.byref(o),
                                      None if out is None else out.ctypes.data_as(vp), mx.ctypes.data_as(pdbl),
                                      mean.ctypes.data_as(pdbl), st.ctypes.data_as(C.POINTER(cint)), C.byref(ms)))
        return out, mx, mean, st, ms.value

    def mc_batch_device(self, p_ptr: int, v_ptr: int, batch: int, opts: BatchOpts, out_ptr: int | None,
                        stats_ptr: int, stream: int | None = None) -> None:
        """Device-resident batch on raw device pointers (e.g. torch .data_ptr())."""
        L = lib()
        # stream None -> library stream; 0 (torch's legacy default stream) -> cudaStreamLegacy (0x1)
        sp = None if stream is None else C.c_void_p(stream if stream else 1)
        check(L, L.gt_mc_batch_device(self._d, C.c_void_p(p_ptr), C.c_void_p(v_ptr), batch, C.byref(opts),
                                      C.c_void_p(out_ptr) if out_ptr else None, C.c_void_p(stats_ptr), sp))

    def fp_opts(self, **kw) -> "FPOpts":
        o = FPOpts()
        lib().gt_fp_opts_default(C.byref(o))
        for k, v in kw.items():
            setattr(o, k, v)
        return o

    def fp_batch_host(self, p_dyn: np.ndarray, var: np.ndarray, opts: "FPOpts | None" = None, t0=None):
        """Mode B from host arrays -> (maps, iters, status, max, ms); t0: initial maps (opts.warm_start)."""
        L = lib()
        dt = np.float64 if self.precision == GT_FP64 else np.float32
        p = np.ascontiguousarray(p_dyn, dtype=dt)
        v = np.ascontiguousarray(var, dtype=dt)
        B = p.shape[0]
        o = opts or self.fp_opts()
        out = np.empty_like(p) if not o.warm_start else np.ascontiguousarray(t0, dtype=dt).copy()
        it = np.empty(B, np.int32)
        st = np.empty(B, np.int32)
        mx = np.empty(B)
        ms = C.c_double()
        check(L, L.gt_fp_batch(self._d, p.ctypes.data_as(vp), v.ctypes.data_as(vp), B, C.byref(o),
                               out.ctypes.data_as(vp), it.ctypes.data_as(C.POINTER(cint)),
                               st.ctypes.data_as(C.POINTER(cint)), mx.ctypes.data_as(pdbl), C.byref(ms)))
        return out, it, st, mx, ms.value

    def fp_batch_device(self, p_ptr, v_ptr, batch, opts, out_ptr, iters_ptr, status_ptr, max_ptr=None,
                        mean_ptr=None, stream=None) -> None:
        L = lib()
        sp = None if stream is None else C.c_void_p(stream if stream else 1)
        check(L, L.gt_fp_batch_device(self._d, C.c_void_p(p_ptr), C.c_void_p(v_ptr), batch, C.byref(opts),
                                      C.c_void_p(out_ptr), C.c_void_p(iters_ptr), C.c_void_p(status_ptr),
                                      C.c_void_p(max_ptr) if max_ptr else None,
                                      C.c_void_p(mean_ptr) if mean_ptr else None, sp))

    def trace_opts(self, **kw) -> "TraceOpts":
        o = TraceOpts()
        lib().gt_trace_opts_default(C.byref(o))
        for k, v in kw.items():
            setattr(o, k, v)
        return o

    def trace_batch_device(self, blk_ptr, blk_stride, sched_ptr, nblk, leak_ptr, leak_stride, batch, opts, out_ptr,
                           max_ptr=None, stream=None) -> None:
        """Config-3 batched traces (include/greentherm_b200.h gt_trace_batch_device); device pointers."""
        L = lib()
        sp = None if stream is None else C.c_void_p(stream if stream else 1)
        check(L, L.gt_trace_batch_device(self._d, C.c_void_p(blk_ptr), blk_stride, C.c_void_p(sched_ptr), nblk,
                                         C.c_void_p(leak_ptr), leak_stride, batch, C.byref(opts),
                                         C.c_void_p(out_ptr), C.c_void_p(max_ptr) if max_ptr else None, sp))

    def profile_begin(self, mode: int = 0) -> None:
        """mode 0: events around all three passes; 1: around the column pass only."""
        check(lib(), lib().gt_profile_begin_mode(self._d, mode))

    def profile_end(self):
        """-> (pass_ms[4], kernels, calls)"""
        ms = (C.c_double * 4)()
        k, c = C.c_longlong(), C.c_longlong()
        check(lib(), lib().gt_profile_end(self._d, ms, C.byref(k), C.byref(c)))
        return list(ms), k.value, c.value
