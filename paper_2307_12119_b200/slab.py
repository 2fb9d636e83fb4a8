"""Config 4: the mode-B fixed point on one large map, slab-decomposed over ranks.

One process per GPU (torch.distributed: NCCL on GPUs; gloo in the CPU tests).
Rank r owns die-row pairs [r P, (r+1) P) (P = n / 2 / world) for the row
phases and half-spectrum columns [c0_r, c0_r + hc_r) for the column phase
(SURVEY §8e). Per iteration:

  rows_fwd (local rows)  -> the rows' spectra: real DCT-II rows [2P][n+1] (n <= 8192:
                            one-pass row kernel) or packed row-pair spectra Z [P][m]
  exchange 1             -> the column phase sees, for ALL row pairs, the
                            columns it owns and their mirrors
  cols (local columns)   -> rows [0, n) of IFFT_col(fk . FFT_col)
  exchange 2             -> every rank gets its rows for all columns
  rows_inv (local rows)  -> theta -> T, residual, next applied rows

Two transports for the exchanges (world > 1):

  "peer" (default on GPUs): no copies. Each rank's Z and row buffer are
      cudaMalloc'ed and mapped into every other rank by CUDA IPC (gt_ipc_*); the
      column kernels read the other ranks' Z in place over NVLink while they
      transform (gt_large_cols_peer: peer loads inside the FFT pass) and store
      each result row straight into its owner's row buffer (peer stores). The
      phases are ordered by a stream sync + barrier after rows_fwd and after cols.
  "nccl": two all_to_all_single calls per iteration on compact per-destination
      blocks (one index_select to pack, one index_copy to unpack): the columns a
      rank owns of every DCT row (or of every packed line plus their mirrors). The
      CPU tests run this path under gloo with numpy stand-in phases, both layouts.

`solve_slab_emulated` runs W ranks' slabs in ONE process on one GPU through the
peer kernels (the rank table holds W same-device buffers) -- the multi-rank data
path exercised without kernels that wait on each other.

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
(`GpuLargeOps`, C ABI gt_large_*); this module only orders phases and moves
blocks between ranks.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from .api import GT_SAMPLE_KIRCHHOFF, GT_SAMPLE_NOCONVERGE, GT_SAMPLE_NONFINITE  # noqa: F401  (header values)


def column_ranges(h: int, world: int) -> list[tuple[int, int]]:
    """Contiguous (c0, hc) per rank covering [0, h), split on even columns: the column
    phase carries columns 2k, 2k+1 on one line, so every rank packs the same pairs as a
    single GPU does (identical bits for any world size)."""
    pairs = (h + 1) // 2
    base, extra = divmod(pairs, world)
    out, p0 = [], 0
    for r in range(world):
        pc = base + (1 if r < extra else 0)
        c0, c1 = 2 * p0, min(h, 2 * (p0 + pc))
        out.append((c0, c1 - c0))
        p0 += pc
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
        lay = C.c_int()
        self._check(self.L.gt_large_row_layout(dg._d, C.byref(lay)))
        self.dct_rows = bool(lay.value)  # rows_fwd writes real DCT rows [2P][n+1] (else packed [P][m])

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

    def cols_peer(self, z_table, world, pairs_per_rank, c0, hc, c1, c2, y_table, hy, stream):
        """z_table / y_table: device int64 tensors of `world` mapped pointers."""
        self._check(self.L.gt_large_cols_peer(self.dg._d, self._p(z_table), world, pairs_per_rank, c0, hc,
                                              self._p(c1), self._p(c2), self._p(y_table), hy, C.c_void_p(stream)))

    # low-mode Anderson mixing on the row buffer (gt_large_lowmode_*: no host synchronisation)
    def lowmode_alloc(self, rows, dev):
        import torch
        nb = self.L.gt_large_lowmode_partial_blocks(rows)
        state = torch.zeros(self.L.gt_large_lowmode_state_bytes(), dtype=torch.uint8, device=dev)
        return (state, torch.empty((nb, 256), dtype=torch.float64, device=dev),
                torch.zeros(256, dtype=torch.float64, device=dev), torch.zeros(256, dtype=torch.float64, device=dev))

    def lowmode_init(self, state, stream):
        self._check(self.L.gt_large_lowmode_init(self._p(state), C.c_void_p(stream)))

    def lowmode_project(self, y, hy, rows, row0, partial, coef, stream):
        self._check(self.L.gt_large_lowmode_project(self.dg._d, self._p(y), hy, rows, row0, self._p(partial),
                                                    self._p(coef), C.c_void_p(stream)))

    def lowmode_mix(self, state, coef, depth, res_prev, corr, stream):
        self._check(self.L.gt_large_lowmode_mix(self._p(state), self._p(coef), depth, float(res_prev),
                                                self._p(corr), C.c_void_p(stream)))

    def lowmode_apply(self, y, hy, rows, row0, corr, stream):
        self._check(self.L.gt_large_lowmode_apply(self.dg._d, self._p(y), hy, rows, row0, self._p(corr),
                                                  C.c_void_p(stream)))

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


class IpcBuffer:
    """A cudaMalloc'ed device buffer with its CUDA IPC handle (gt_ipc_alloc), viewed as a
    torch tensor (zero copy, __cuda_array_interface__); `open_peer` maps another rank's."""

    def __init__(self, shape, dtype, device):
        import torch
        from .api import check, lib
        self.L = lib()
        self.shape, self.dtype = tuple(shape), dtype
        nbytes = int(np.prod(shape)) * torch.empty((), dtype=dtype).element_size()
        self.ptr = C.c_void_p()
        self.handle = (C.c_char * 64)()
        check(self.L, self.L.gt_ipc_alloc(nbytes, C.byref(self.ptr), self.handle))
        self.tensor = _wrap(self.ptr.value, self.shape, dtype, device)

    def handle_bytes(self) -> bytes:
        return bytes(self.handle)

    def close(self):
        if self.ptr:
            self.tensor = None
            self.L.gt_ipc_free(self.ptr)
            self.ptr = C.c_void_p()


def open_peer(handle: bytes) -> int:
    from .api import check, lib
    L = lib()
    buf = (C.c_char * 64).from_buffer_copy(handle)
    p = C.c_void_p()
    check(L, L.gt_ipc_open(buf, C.byref(p)))
    return p.value


def _wrap(ptr, shape, dtype, device):
    """Zero-copy torch view of a raw device pointer."""
    import torch
    typestr = {torch.float64: "<f8", torch.complex128: "<c16", torch.int64: "<i8"}[dtype]

    class _Arr:
        __cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (ptr, False), "version": 3,
                                    "strides": None}
    return torch.as_tensor(_Arr(), device=device)


@dataclass
class SlabResult:
    t: "object"          # local rows of the converged rise map [2P][n]
    iterations: int
    status: int
    residual: float


class _Accel:
    """Chebyshev omega / gamma schedule from the residual history (fixed_point.cu fp_update)."""

    def __init__(self, k0):
        self.k0 = k0
        self.omega, self.gamma, self.sigma2, self.res_prev = 0.0, 1.0, 0.0, 0.0

    def update(self, it, res):
        if self.k0 <= 0:
            return
        if self.omega > 0.0:
            if res > 2.0 * self.res_prev:
                self.omega, self.gamma = -1.0, 1.0  # diverging under acceleration: plain Picard from here on
            else:
                self.omega = (2.0 / (2.0 - self.sigma2) if self.omega == 1.0
                              else 1.0 / (1.0 - 0.25 * self.sigma2 * self.omega))
        elif self.omega == 0.0 and it == self.k0 and self.res_prev > 0.0:
            rho = min(0.97, max(0.0, 1.02 * res / self.res_prev))
            self.gamma = 2.0 / (2.0 - rho)
            self.sigma2 = (rho / (2.0 - rho)) ** 2
            self.omega = 1.0
        self.res_prev = res


class _LowMode:
    """Anderson(m) mixing on the K x K lowest cosine modes of the die field (opts.accel = -m;
    the batched path's fp_lowmode kernel, fixed_point.cu), applied to the row buffer Y between
    the column phase and the inverse row phase. A mirrored row with cosine content d_q has
    Y[q] = conj(hs_q) M^2 eps_q d_q (hs_q = exp(-i pi q / m), eps_0 = 1, eps_q = 1/2), so the
    coefficients are a_pq = sum_x cos(pi p (x + 1/2) / n) Re(hs_q Y[x][q]) / (M^2 eps_q n eps_p)
    -- partial sums over this rank's rows, all-reduced (256 doubles) -- and the correction is
    added back to the same 16 columns. The 256-dimensional least squares runs on the host."""
    K = 16

    def __init__(self, depth, n, rows, row0, dev, world, ops=None, stream=0):
        import numpy as np
        import torch
        self.depth, self.n, self.world = depth, n, world
        self.rows, self.row0, self.stream = rows, row0, stream
        # device kernels when the ops provide them (GpuLargeOps); the torch / numpy
        # restatement below serves the CPU stand-in ops of the gloo tests
        self.ops = ops if (ops is not None and hasattr(ops, "lowmode_project") and dev.type == "cuda") else None
        if self.ops is not None:
            self.state, self.partial, self.coef, self.corr = self.ops.lowmode_alloc(rows, dev)
            self.ops.lowmode_init(self.state, stream)
            self.rprev_seen = 0.0
            return
        K, m = self.K, 2 * n
        q = torch.arange(K, device=dev, dtype=torch.float64)
        x = torch.arange(row0, row0 + rows, device=dev, dtype=torch.float64)
        self.cos = torch.cos(torch.pi * q[:, None] * (x[None, :] + 0.5) / n).contiguous()  # [K(p)][rows]
        self.hs = torch.polar(torch.ones_like(q), -torch.pi * q / m)                        # [K] exp(-i pi q / m)
        eps = torch.full((K,), 0.5, dtype=torch.float64, device=dev)
        eps[0] = 1.0
        self.scale_q = (float(m) * float(m)) * eps                                         # [K(q)]
        self.norm = 1.0 / (self.scale_q[None, :] * (n * eps)[:, None])                     # [K(p)][K(q)]
        self.xlow = np.zeros(K * K)
        self.gprev = self.fprev = None
        self.dG, self.dF = [], []
        self.calls, self.rprev = 0, 0.0

    def project(self, y):
        """Partial coefficients [K(p)][K(q)] from this rank's rows of the row buffer."""
        K = self.K
        d = (self.hs[None, :] * y[:, :K]).real                      # [rows][K(q)]
        return (self.cos @ d) * self.norm

    def mix(self, a, res_prev):
        """Anderson step on the summed coefficients `a`; returns the correction [K][K] (numpy)
        or None. res_prev: the residual of the previous iteration (growth guard)."""
        import numpy as np
        K = self.K
        g = a.detach().cpu().numpy().reshape(-1).copy()
        if self.calls > 1 and self.rprev > 0.0 and res_prev > 2.0 * self.rprev:
            self.dG, self.dF = [], []                               # residual doubled: drop the history
            self.gprev = None
        f = g - self.xlow
        if self.gprev is not None:
            self.dG.append(g - self.gprev)
            self.dF.append(f - self.fprev)
            self.dG, self.dF = self.dG[-self.depth:], self.dF[-self.depth:]
        self.gprev, self.fprev = g, f
        corr = np.zeros_like(g)
        if self.dF:
            A = np.stack(self.dF, 1)
            gram = A.T @ A
            tr = float(np.trace(gram))
            if tr > 0.0:
                gam = np.linalg.solve(gram + 1e-10 * tr * np.eye(gram.shape[0]), A.T @ f)
                if np.all(np.isfinite(gam)) and np.abs(gam).max() <= 1e3:
                    corr = -(np.stack(self.dG, 1) @ gam)
                else:
                    self.dG, self.dF = [], []
        self.xlow = g + corr
        self.calls += 1
        self.rprev = res_prev
        return corr.reshape(K, K) if np.any(corr) else None

    def apply(self, y, corr):
        """Add the correction's row spectra to columns q < K of this rank's rows (in place)."""
        import torch
        if corr is None:
            return
        c = torch.from_numpy(corr).to(y.device)
        add = (self.cos.T @ c) * self.scale_q[None, :]               # [rows][K(q)]
        y[:, :self.K] += torch.conj(self.hs)[None, :] * add

    def step(self, y, res_prev):
        """y: this rank's row buffer [rows][hy] complex128, corrected in place."""
        import math
        import torch.distributed as dist
        if self.ops is not None:
            hy = y.stride(0)
            self.ops.lowmode_project(y, hy, self.rows, self.row0, self.partial, self.coef, self.stream)
            if self.world > 1:
                if dist.get_backend() == "nccl":
                    dist.all_reduce(self.coef)
                else:  # gloo (tests): through the host
                    c = self.coef.cpu()
                    dist.all_reduce(c)
                    self.coef.copy_(c)
            rp = res_prev if math.isfinite(res_prev) else 0.0
            self.ops.lowmode_mix(self.state, self.coef, self.depth, rp, self.corr, self.stream)
            self.ops.lowmode_apply(y, hy, self.rows, self.row0, self.corr, self.stream)
            return
        a = self.project(y)
        if self.world > 1:
            if dist.get_backend() != "nccl":
                a = a.cpu()
            dist.all_reduce(a)
        self.apply(y, self.mix(a, res_prev))


class _RankState:
    """One rank's slab: rows [2P][n], its spectra / scratch buffers and loop state."""

    def __init__(self, n, P, c0, hc, p_local, v_local, opts, z=None, yrow=None):
        import torch
        dev = p_local.device
        m, h = 2 * n, n + 1
        cd = torch.complex128
        self.P, self.c0, self.hc = P, c0, hc
        self.p = p_local
        self.l0 = opts.leak_frac * p_local * v_local
        self.app = (p_local + self.l0).contiguous()
        self.t = torch.zeros_like(p_local)
        self.s1 = torch.empty((P, m), dtype=cd, device=dev)
        self.z = z if z is not None else torch.empty((P, m), dtype=cd, device=dev)
        self.c1 = torch.empty((m, hc), dtype=cd, device=dev)
        self.c2 = torch.empty((m, hc), dtype=cd, device=dev)
        self.yrow = yrow  # [2P][h] row buffer (peer / nccl transports)
        self.res_bits = torch.zeros(1, dtype=torch.int64, device=dev)
        self.status = torch.zeros(1, dtype=torch.int32, device=dev)
        accel = int(getattr(opts, "accel", 0) or 0)
        self.q = torch.zeros_like(p_local) if accel > 0 else None  # x_{k-1} in, x_k out
        self.g = torch.empty_like(p_local) if accel > 0 else None  # G(x_k)

    def rows_inv(self, ops, y, hy, opts, acc, stream):
        self.res_bits.zero_()
        ops.rows_inv(y, hy, self.P, self.s1, self.t, self.app, self.p, self.l0, opts, self.res_bits, self.status,
                     stream, q=self.q, g=self.g, omega=max(acc.omega, 0.0), gamma=acc.gamma)

    def finish(self):
        if self.g is not None:
            self.t.copy_(self.g)  # G(x_k): its error bound is the stop rule's, not that of the extrapolated x_{k+1}


def _stop(it, res, st, opts, acc):
    """Reference stop rule after iteration `it`; returns (done, status)."""
    if st:
        return True, st
    acc.update(it, res)
    if it > 1 and res < opts.tol:
        return True, st
    if it == opts.max_iters:
        return True, st | GT_SAMPLE_NOCONVERGE
    return False, st


def solve_slab(ops, n: int, p_local, v_local, opts, rank: int = 0, world: int = 1, stream: int | None = None,
               exchange=None, transport: str | None = None) -> SlabResult:
    """Fixed point on the local slab. p_local / v_local: [2P][n] float64 tensors of
    this rank's rows; opts: api.FPOpts (leak_frac, law, kirchhoff, beta, t_ambient,
    eta, tol, max_iters, accel). Device work is issued on `stream` (default: torch's
    current stream, which the NCCL exchange also uses). transport: "peer" (CUDA IPC
    mapped buffers, default for CUDA tensors) or "nccl" (all-to-all copies; `exchange`
    defaults to torch.distributed.all_to_all_single and is injectable for tests)."""
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
    if transport is None:
        transport = "peer" if (dev.type == "cuda" and exchange is None and world > 1) else "nccl"
    if stream is None:
        stream = torch.cuda.current_stream(dev).cuda_stream if dev.type == "cuda" else 0
    cd = torch.complex128
    acc = _Accel(int(getattr(opts, "accel", 0) or 0))
    ipc = []
    if world > 1 and transport == "peer":
        zb = IpcBuffer((P, m), cd, dev)
        yb = IpcBuffer((rows, h), cd, dev)
        ipc = [zb, yb]
        S = _RankState(n, P, c0, hc, p_local, v_local, opts, z=zb.tensor, yrow=yb.tensor)
        handles = [None] * world
        dist.all_gather_object(handles, (zb.handle_bytes(), yb.handle_bytes()))
        opened = []
        zp, yp = [], []
        for r, (hz, hy_) in enumerate(handles):
            if r == rank:
                zp.append(zb.ptr.value)
                yp.append(yb.ptr.value)
            else:
                a, b = open_peer(hz), open_peer(hy_)
                opened += [a, b]
                zp.append(a)
                yp.append(b)
        z_table = torch.tensor(zp, dtype=torch.int64, device=dev)
        y_table = torch.tensor(yp, dtype=torch.int64, device=dev)
    else:
        S = _RankState(n, P, c0, hc, p_local, v_local, opts)
    exchange = exchange or (dist.all_to_all_single if world > 1 else None)
    dct = bool(getattr(ops, "dct_rows", False))
    if world > 1 and transport == "nccl":
        ycol = torch.empty((n, hc), dtype=cd, device=dev)
        S.yrow = torch.empty((rows, h), dtype=cd, device=dev)
        # Per-destination send blocks as ONE gather from the row phase's output: block q holds,
        # for every local row, the columns rank q owns (DCT rows [rows][h], real), or, packed,
        # for every local row pair those columns and their mirrors m - v (compact layouts of
        # gt_large_cols). The index maps are built once; each iteration is a single
        # index_select into a preallocated buffer (no per-iteration concatenation).
        cols = []
        for cq, hq in ranges:
            own = torch.arange(cq, cq + hq, device=dev)
            if dct:
                cols.append((torch.arange(rows, device=dev)[:, None] * h + own[None, :]).reshape(-1))
            else:
                blk = torch.cat([own, torch.remainder(m - own, m)])
                cols.append((torch.arange(P, device=dev)[:, None] * m + blk[None, :]).reshape(-1))
        send_idx = torch.cat(cols)
        zdt = torch.float64 if dct else cd
        send = torch.empty(send_idx.numel(), dtype=zdt, device=dev)
        zrecv = (torch.empty((world, rows, hc), dtype=zdt, device=dev) if dct
                 else torch.empty((world, P, 2 * hc), dtype=cd, device=dev))
        # receive side of the second exchange: source q's block [rows][hq] lands in columns
        # [cq, cq + hq) of yrow -- one index_copy with a precomputed destination map
        dst = [(torch.arange(rows, device=dev)[:, None] * h + torch.arange(cq, cq + hq, device=dev)[None, :])
               .reshape(-1) for cq, hq in ranges]
        recv_dst = torch.cat(dst)
        recv = torch.empty(recv_dst.numel(), dtype=cd, device=dev)
    elif world == 1:
        ycol = torch.empty((n, hc), dtype=cd, device=dev)

    def phase_barrier():
        # every rank's previous phase has completed on its GPU before any rank starts the next
        torch.cuda.synchronize(dev)
        dist.barrier()

    it, res, st = 0, float("inf"), 0
    lm_depth = -int(getattr(opts, "accel", 0) or 0)
    lowmode = (_LowMode(min(lm_depth, 4), n, rows, rank * rows, dev, world, ops=ops, stream=stream)
               if lm_depth > 0 and n >= _LowMode.K else None)
    try:
        for it in range(1, opts.max_iters + 1):
            ops.rows_fwd(S.app, P, S.s1, S.z, stream)
            if world == 1:
                ops.cols(S.z, False, c0, hc, S.c1, S.c2, ycol, stream)
                yrow_t = ycol
            elif transport == "peer":
                phase_barrier()  # all row spectra written
                ops.cols_peer(z_table, world, P, c0, hc, S.c1, S.c2, y_table, h, stream)
                phase_barrier()  # all column results stored into their owners' row buffers
                yrow_t = S.yrow
            else:
                zsrc = S.z.view(-1).view(torch.float64)[: rows * h] if dct else S.z.view(-1)
                torch.index_select(zsrc, 0, send_idx, out=send)
                # output splits: what each source sends me; input splits: what I send each rank.
                # Complex blocks travel as their float64 (re, im) view (NCCL has no complex type).
                if dct:
                    exchange(zrecv.view(-1), send, [rows * hc] * world, [rows * hq for _, hq in ranges])
                    ops.cols(zrecv.reshape(n, hc), True, c0, hc, S.c1, S.c2, ycol, stream)
                else:
                    exchange(torch.view_as_real(zrecv).view(-1), torch.view_as_real(send).view(-1),
                             [2 * P * 2 * hc] * world, [2 * P * 2 * hq for _, hq in ranges])
                    ops.cols(zrecv.reshape(n // 2, 2 * hc), True, c0, hc, S.c1, S.c2, ycol, stream)
                # ycol [n][hc] is already [world][rows][hc]: rank q's rows are a contiguous block
                exchange(torch.view_as_real(recv).view(-1), torch.view_as_real(ycol).view(-1),
                         [2 * rows * hq for _, hq in ranges], [2 * rows * hc] * world)
                S.yrow.view(-1).index_copy_(0, recv_dst, recv)
                yrow_t = S.yrow
            if lowmode is not None:
                lowmode.step(yrow_t, res)
            S.rows_inv(ops, yrow_t, h, opts, acc, stream)
            rs = torch.stack([S.res_bits.view(torch.float64)[0], S.status.to(torch.float64)[0]])
            if world > 1 and dist.get_backend() != "nccl":
                rs = rs.cpu()  # gloo gathers host tensors
            if world > 1:
                flags = [torch.zeros_like(rs) for _ in range(world)]
                dist.all_gather(flags, rs)
                res = max(float(f[0]) for f in flags)
                st = 0
                for f in flags:
                    st |= int(f[1])
            else:
                res, st = float(rs[0]), int(rs[1])
            done, st = _stop(it, res, st, opts, acc)
            if done:
                break
        S.finish()
    finally:
        if ipc:
            torch.cuda.synchronize(dev)
            dist.barrier()  # no rank still reads a buffer another rank is about to free
            from .api import lib
            for p in opened:
                lib().gt_ipc_close(C.c_void_p(p))
            S.z = S.yrow = None
            for b in ipc:
                b.close()
    return SlabResult(t=S.t, iterations=it, status=st, residual=res)


def solve_slab_emulated(ops, n: int, p_full, v_full, opts, world: int, stream: int | None = None) -> SlabResult:
    """`world` ranks' slabs in ONE process on one GPU through the peer column kernels
    (gt_large_cols_peer reads every rank's Z in place and stores into every rank's row
    buffer; the rank tables hold same-device pointers). Each phase runs for all ranks
    before the next starts, so no kernel waits on another. Returns the full map."""
    import torch
    if (n // 2) % world:
        raise ValueError("world size must divide n / 2 (whole row pairs per rank)")
    dev = p_full.device
    m, h = 2 * n, n + 1
    P = (n // 2) // world
    rows = 2 * P
    ranges = column_ranges(h, world)
    if stream is None:
        stream = torch.cuda.current_stream(dev).cuda_stream
    cd = torch.complex128
    R = [_RankState(n, P, c0, hc, p_full[r * rows:(r + 1) * rows].contiguous(),
                    v_full[r * rows:(r + 1) * rows].contiguous(), opts,
                    yrow=torch.empty((rows, h), dtype=cd, device=dev))
         for r, (c0, hc) in enumerate(ranges)]
    z_table = torch.tensor([s.z.data_ptr() for s in R], dtype=torch.int64, device=dev)
    y_table = torch.tensor([s.yrow.data_ptr() for s in R], dtype=torch.int64, device=dev)
    acc = _Accel(int(getattr(opts, "accel", 0) or 0))
    lm_depth = -int(getattr(opts, "accel", 0) or 0)
    lms = ([_LowMode(min(lm_depth, 4), n, rows, r * rows, dev, 1) for r in range(world)]
           if lm_depth > 0 and n >= _LowMode.K else [])
    it, res, st = 0, float("inf"), 0
    for it in range(1, opts.max_iters + 1):
        for s in R:
            ops.rows_fwd(s.app, P, s.s1, s.z, stream)
        for s in R:
            ops.cols_peer(z_table, world, P, s.c0, s.hc, s.c1, s.c2, y_table, h, stream)
        if lms:
            corr = lms[0].mix(sum(lm.project(s.yrow) for lm, s in zip(lms, R)), res)
            for lm, s in zip(lms, R):
                lm.apply(s.yrow, corr)
        for s in R:
            s.rows_inv(ops, s.yrow, h, opts, acc, stream)
        res = max(float(s.res_bits.view(torch.float64)[0]) for s in R)
        st = 0
        for s in R:
            st |= int(s.status[0])
        done, st = _stop(it, res, st, opts, acc)
        if done:
            break
    for s in R:
        s.finish()
    return SlabResult(t=torch.cat([s.t for s in R]), iterations=it, status=st, residual=res)
