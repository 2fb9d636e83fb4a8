"""TEST INFRASTRUCTURE: numpy stand-ins for the three device phases of
paper_2307_12119_b200/slab.py (same buffer layouts as the gt_large_* kernels),
so the slab exchange logic can run on CPU ranks under gloo."""
import numpy as np


class NumpyLargeOps:
    def __init__(self, n, fk, dct_rows=False):
        self.n, self.m = n, 2 * n
        self.fk = fk  # [m][m] complex, full baseline kernel spectrum
        # dct_rows: rows_fwd writes the rows' real DCT-II coefficients [rows][n+1] (the device
        # layout for n <= 8192); else the packed row-pair spectra [pairs][m]
        self.dct_rows = dct_rows
        self.hs = np.exp(-1j * np.pi * np.arange(self.m) / self.m)

    def _mirror(self):
        i = np.arange(self.m)
        return np.where(i < self.n, i, self.m - 1 - i)

    def rows_fwd(self, app, pairs, s1, z, stream):
        a = app.numpy()
        mi = self._mirror()
        if self.dct_rows:
            h = self.n + 1
            at = z.view(-1).view(__import__("torch").float64).numpy()
            for x in range(2 * pairs):
                U = np.fft.fft(a[x][mi])[:h]
                at[x * h:(x + 1) * h] = np.real(self.hs[:h] * U)
            return
        for p in range(pairs):
            x = a[2 * p][mi] + 1j * a[2 * p + 1][mi]
            z[p] = __import__("torch").from_numpy(np.fft.fft(x))

    def cols(self, z, compact, c0, hc, c1, c2, y, stream):
        n, m = self.n, self.m
        Z = z.numpy()
        mi = self._mirror()
        out = np.zeros((n, hc), complex)
        if self.dct_rows:
            At = z.numpy().reshape(n, hc) if compact else z.view(-1).view(__import__("torch").float64).numpy()[
                : n * (n + 1)].reshape(n, n + 1)[:, c0:c0 + hc]
        for c in range(hc):
            v = c0 + c
            if self.dct_rows:
                A = np.conj(self.hs[v]) * At[:, c]
            else:
                if compact:
                    a, b = Z[:, c], np.conj(Z[:, hc + c])
                else:
                    a, b = Z[:, v], np.conj(Z[:, (m - v) % m])
                A = np.empty(n, complex)
                A[0::2] = 0.5 * (a + b)
                A[1::2] = -0.5j * (a - b)
            col = np.fft.fft(A[mi])
            col = col * self.fk[:, v] if v <= n else col * 0
            out[:, c] = (np.fft.ifft(col) * m)[:n]
        y.copy_(__import__("torch").from_numpy(out))

    def rows_inv(self, y, hy, pairs, s1, t, app, p, l0, opts, res_bits, status, stream, q=None, g=None,
                 omega=0.0, gamma=1.0):
        import torch
        n, m = self.n, self.m
        Y = y.numpy()
        T, A, Pm, L = t.numpy(), app.numpy(), p.numpy(), l0.numpy()
        f = np.arange(m)
        w = np.where(f <= n, f, m - f)
        dmax = 0.0
        for pq in range(pairs):
            r0, r1 = Y[2 * pq][w], Y[2 * pq + 1][w]
            r0 = np.where(f <= n, r0, np.conj(r0))
            r1 = np.where(f <= n, r1, np.conj(r1))
            line = (np.fft.ifft(r0 + 1j * r1) * m)[:n] / (m * m)
            for half, th in ((0, line.real), (1, line.imag)):
                x = 2 * pq + half
                tt = th
                if opts.kirchhoff:
                    a_ = opts.t_ambient ** (1 - opts.eta)
                    b_ = (1 - opts.eta) * opts.t_ambient ** (-opts.eta)
                    tt = (a_ + b_ * th) ** (1 / (1 - opts.eta)) - opts.t_ambient
                dmax = max(dmax, float(np.abs(tt - T[x]).max()))
                if g is not None:
                    g.numpy()[x] = tt
                if q is not None:
                    Q = q.numpy()
                    xprev = Q[x].copy()
                    Q[x] = T[x]
                    if omega > 0:
                        tt = omega * (gamma * tt + (1 - gamma) * T[x] - xprev) + xprev
                T[x] = tt
                fl = 1 + opts.beta * tt if opts.law == 0 else np.exp(opts.beta * tt)
                A[x] = Pm[x] + L[x] * fl
        cur = res_bits.view(torch.float64)
        cur[0] = max(float(cur[0]), dmax)


def baseline_fk(f_sp0, phi):
    """fk = FFT2(center_kernel(f_sp0 - phi)); fk[0,0] += phi m^2 / 4 (reference greens.cpp:194-201)."""
    n = f_sp0.shape[0]
    m, c = 2 * n, n // 2
    K = np.zeros((m, m))
    x = (np.arange(n) - c) % m
    K[np.ix_(x, x)] = f_sp0 - phi
    fk = np.fft.fft2(K)
    fk[0, 0] += phi * m * m / 4
    return fk


def fixed_point_numpy(P, V, fk, leak_frac, beta, law, tol, max_iters):
    """Direct 2-D restatement of the loop (crop(IFFT2(fk . FFT2(mirror(applied)))))."""
    n = P.shape[0]
    m = 2 * n
    mi = np.where(np.arange(m) < n, np.arange(m), m - 1 - np.arange(m))
    L0 = leak_frac * P * V
    T = np.zeros_like(P)
    for it in range(1, max_iters + 1):
        app = P + L0 * (1 + beta * T if law == 0 else np.exp(beta * T))
        th = np.fft.ifft2(fk * np.fft.fft2(app[np.ix_(mi, mi)])).real[:n, :n]
        d = np.abs(th - T).max()
        T = th
        if it > 1 and d < tol:
            return T, it
    return T, max_iters


def fixed_point_torch(P, V, f_sp0, phi, leak_frac, beta, law, tol, max_iters):
    """fixed_point_numpy on the GPU in fp64 (torch.fft, test-side checker for n = 8192):
    T_{k+1} = crop(IRFFT2(fk . RFFT2(mirror(P + L0 f(T_k))))), fk = FFT2(center_kernel(f_sp0 - phi))
    + phi m^2/4 at DC (greens.cpp:194-201), stop when max|dT| < tol after iteration 1."""
    import torch
    n = P.shape[0]
    m, c = 2 * n, n // 2
    dev = P.device
    K = torch.zeros((m, m), dtype=torch.float64, device=dev)
    x = (torch.arange(n, device=dev) - c) % m
    K[x[:, None], x[None, :]] = f_sp0 - phi
    fk = torch.fft.rfft2(K)
    del K
    fk[0, 0] += phi * m * m / 4
    L0 = leak_frac * P * V
    T = torch.zeros_like(P)
    for it in range(1, max_iters + 1):
        app = P + L0 * (1 + beta * T if law == 0 else torch.exp(beta * T))
        mir = torch.cat([app, app.flip(0)], 0)
        mir = torch.cat([mir, mir.flip(1)], 1)
        th = torch.fft.irfft2(fk * torch.fft.rfft2(mir), s=(m, m))[:n, :n]
        d = float((th - T).abs().max())
        T = th.contiguous()
        if it > 1 and d < tol:
            return T, it
    return T, max_iters
