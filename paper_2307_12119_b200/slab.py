"""Config 4: the mode-B fixed point on one large map, slab-decomposed over ranks.

One process per GPU (torch.distributed, NCCL on GPUs; gloo in the CPU tests).
Rank r owns die-row pairs [r P, (r+1) P) (P = n / 2 / world) for the row
phases and half-spectrum columns [c0_r, c0_r + hc_r) for the column phase
(SURVEY §8e). Per iteration:

  rows_fwd (local rows)  -> Z [P][m]   spectra of the mirrored row pairs
  all-to-all             -> every rank gets, for ALL row pairs, the columns it
                            owns and their mirrors (compact [n/2][2 hc] layout)
  cols (local columns)   -> Y [n][hc]  rows [0, n) of IFFT_col(fk . FFT_col)
  all-to-all             -> every rank gets its rows for all columns
  rows_inv (local rows)  -> theta -> T, residual, next applied rows

The stop rule is the reference outer loop's (fdm.cpp:190-200): converged when
max|T_{k+1} - T_k| < tol after iteration 1 (max over ranks), max_iters ->
GT_SAMPLE_NOCONVERGE. With world = 1 no exchange happens and the column phase
reads the row spectra in place.

opts.accel = k0 > 0 runs the Chebyshev semi-iteration of gt_fp_batch (fixed_point.cu
fp_update) on the same Picard map: plain iterations up to k0, the contraction rate
rho from the residual ratio there (max over ranks, so every rank takes the same
steps), then x_{k+1} = omega (gamma G(x_k) + (1 - gamma) x_k - x_{k-1}) + x_{k-1}
in the inverse row pass; a residual that doubles falls back to Picard. The stop
rule is unchanged (max|G(x_k) - x_k| < tol) and the result is G(x_k).

The arithmetic lives in the sm_100a passes of libgreentherm_b200.so
(`GpuLargeOps`, C ABI gt_large_*); this module only moves blocks between ranks.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from .api import GT_SAMPLE_KIRCHHOFF, GT_SAMPLE_NOCONVERGE, GT_SAMPLE_NONFINITE  # noqa: F401  (header values)


def column_ranges(h: int, world: int) -> list[tuple[int, int]]:
    """Contiguous (c0, hc) per rank covering [0, h)."""
    base, extra = divmod(h, world)
    out, c0 = [], 0
    for r in range(world):
        hc = base + (1 if r < extra else 0)
        out.append((c0, hc))
        c0 += hc
    return out


class GpuLargeOps:
    """The three phases on the device (C ABI gt_large_*; torch CUDA tensors)."""

    def __init__(self, dg):
        from .api import lib
        self.L = lib()
        self.dg = dg
        m1, m2 = C.c_int(), C.c_int()
        self._check(self.L.gt_large_geometry(dg._d, C.byref(m1), C.byref(m2)))
        self.M1, self.M2 = m1.value, m2.value

    def _check(self, st):
        from .api import check
        check(self.L, st)

    @staticmethod
    def _p(t):
        return C.c_void_p(t.data_ptr())

    def rows_fwd(self, app, pairs, s1, z, stream):
        self._check(self.L.gt_large_rows_fwd(self.dg._d, self._p(app), pairs, self._p(s1), self._p(z),
                                             C.c_void_p(stream)))

    def cols(self, z, compact, c0, hc, c1, c2, y, stream):
        self._check(self.L.gt_large_cols(self.dg._d, self._p(z), int(compact), c0, hc, self._p(c1), self._p(c2),
                                         self._p(y), C.c_void_p(stream)))

    def rows_inv(self, y, hy, pairs, s1, t, app, p, l0, opts, res_bits, status, stream, q=None, g=None,
                 omega=0.0, gamma=1.0):
        if q is None:
            self._check(self.L.gt_large_rows_inv(self.dg._d, self._p(y), hy, pairs, self._p(s1), self._p(t),
                                                 self._p(app), self._p(p), self._p(l0), C.byref(opts),
                                                 self._p(res_bits), self._p(status), C.c_void_p(stream)))
        else:
            self._check(self.L.gt_large_rows_inv_accel(
                self.dg._d, self._p(y), hy, pairs, self._p(s1), self._p(t), self._p(app), self._p(p), self._p(l0),
                C.byref(opts), self._p(res_bits), self._p(status), self._p(q), self._p(g), float(omega),
                float(gamma), C.c_void_p(stream)))


@dataclass
class SlabResult:
    t: "object"          # local rows of the converged rise map [2P][n]
    iterations: int
    status: int
    residual: float


def solve_slab(ops, n: int, p_local, v_local, opts, rank: int = 0, world: int = 1, stream: int | None = None,
               exchange=None) -> SlabResult:
    """Fixed point on the local slab. p_local / v_local: [2P][n] float64 tensors of
    this rank's rows; opts: api.FPOpts (leak_frac, law, kirchhoff, beta, t_ambient,
    eta, tol, max_iters). Device work is issued on `stream` (default: torch's
    current stream, which the NCCL exchange also uses). `exchange` (default
    torch.distributed.all_to_all_single) is injectable for tests."""
    import torch
    import torch.distributed as dist
    if (n // 2) % world:
        raise ValueError("world size must divide n / 2 (whole row pairs per rank)")
    dev = p_local.device
    m, h = 2 * n, n + 1
    P = (n // 2) // world
    rows = 2 * P
    ranges = column_ranges(h, world)
    c0, hc = ranges[rank]
    exchange = exchange or dist.all_to_all_single
    if stream is None:
        stream = torch.cuda.current_stream(dev).cuda_stream if dev.type == "cuda" else 0
    cd = torch.complex128
    l0 = opts.leak_frac * p_local * v_local
    app = (p_local + l0).contiguous()
    t = torch.zeros_like(p_local)
    s1 = torch.empty((P, m), dtype=cd, device=dev)
    z = torch.empty((P, m), dtype=cd, device=dev)
    c1 = torch.empty((m, hc), dtype=cd, device=dev)
    c2 = torch.empty((m, hc), dtype=cd, device=dev)
    ycol = torch.empty((n, hc), dtype=cd, device=dev)
    accel = int(getattr(opts, "accel", 0) or 0)
    q = torch.zeros_like(p_local) if accel > 0 else None  # x_{k-1} in, x_k out
    g = torch.empty_like(p_local) if accel > 0 else None  # G(x_k)
    omega, gamma, sigma2, res_prev = 0.0, 1.0, 0.0, 0.0
    res_bits = torch.zeros(1, dtype=torch.int64, device=dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    if world > 1:
        zrecv = torch.empty((world, P, 2 * hc), dtype=cd, device=dev)
        yrow = torch.empty((rows, h), dtype=cd, device=dev)
        # Per-destination send blocks as ONE gather from the row spectra z [P][m]: block q holds,
        # for every local row pair, the columns rank q owns and their mirrors m - v (compact
        # layout of gt_large_cols). The index maps are built once; each iteration is a single
        # index_select into a preallocated buffer (no per-iteration concatenation).
        cols = []
        for cq, hq in ranges:
            own = torch.arange(cq, cq + hq, device=dev)
            blk = torch.cat([own, torch.remainder(m - own, m)])
            cols.append((torch.arange(P, device=dev)[:, None] * m + blk[None, :]).reshape(-1))
        send_idx = torch.cat(cols)
        send = torch.empty(send_idx.numel(), dtype=cd, device=dev)
        # receive side of the second exchange: source q's block [rows][hq] lands in columns
        # [cq, cq + hq) of yrow -- one index_copy with a precomputed destination map
        dst = [(torch.arange(rows, device=dev)[:, None] * h + torch.arange(cq, cq + hq, device=dev)[None, :])
               .reshape(-1) for cq, hq in ranges]
        recv_dst = torch.cat(dst)
        recv = torch.empty(recv_dst.numel(), dtype=cd, device=dev)
    it, res, st = 0, float("inf"), 0
    for it in range(1, opts.max_iters + 1):
        ops.rows_fwd(app, P, s1, z, stream)
        if world == 1:
            ops.cols(z, False, c0, hc, c1, c2, ycol, stream)
            yrow_t, hy = ycol, h
        else:
            torch.index_select(z.view(-1), 0, send_idx, out=send)
            # output splits: what each source sends me; input splits: what I send each rank.
            # Complex blocks travel as their float64 (re, im) view (NCCL has no complex type).
            exchange(torch.view_as_real(zrecv).view(-1), torch.view_as_real(send).view(-1),
                     [2 * P * 2 * hc] * world, [2 * P * 2 * hq for _, hq in ranges])
            ops.cols(zrecv.reshape(n // 2, 2 * hc), True, c0, hc, c1, c2, ycol, stream)
            # ycol [n][hc] is already [world][rows][hc]: rank q's rows are a contiguous block
            exchange(torch.view_as_real(recv).view(-1), torch.view_as_real(ycol).view(-1),
                     [2 * rows * hq for _, hq in ranges], [2 * rows * hc] * world)
            yrow.view(-1).index_copy_(0, recv_dst, recv)
            yrow_t, hy = yrow, h
        res_bits.zero_()
        ops.rows_inv(yrow_t, hy, P, s1, t, app, p_local, l0, opts, res_bits, status, stream, q=q, g=g,
                     omega=max(omega, 0.0), gamma=gamma)
        rs = torch.stack([res_bits.view(torch.float64)[0], status.to(torch.float64)[0]])
        if world > 1:
            flags = [torch.zeros_like(rs) for _ in range(world)]
            dist.all_gather(flags, rs)
            res = max(float(f[0]) for f in flags)
            st = 0
            for f in flags:
                st |= int(f[1])
        else:
            res, st = float(rs[0]), int(rs[1])
        if st:
            break
        if accel > 0:  # the next step's omega (fixed_point.cu fp_update)
            if omega > 0.0:
                if res > 2.0 * res_prev:
                    omega, gamma = -1.0, 1.0  # diverging under acceleration: plain Picard from here on
                else:
                    omega = 2.0 / (2.0 - sigma2) if omega == 1.0 else 1.0 / (1.0 - 0.25 * sigma2 * omega)
            elif omega == 0.0 and it == accel and res_prev > 0.0:
                rho = min(0.97, max(0.0, 1.02 * res / res_prev))
                gamma = 2.0 / (2.0 - rho)
                sigma2 = (rho / (2.0 - rho)) ** 2
                omega = 1.0
            res_prev = res
        if it > 1 and res < opts.tol:
            break
        if it == opts.max_iters:
            st |= GT_SAMPLE_NOCONVERGE
    if accel > 0:
        t.copy_(g)  # G(x_k): its error bound is the stop rule's, not that of the extrapolated x_{k+1}
    return SlabResult(t=t, iterations=it, status=st, residual=res)
