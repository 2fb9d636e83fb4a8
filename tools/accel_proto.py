"""CPU prototype (numpy, fp64): iterations of the mode-B fixed point on config-1 pairs for
Picard, Chebyshev (start k0) and Anderson(m) acceleration; the count is the number of Picard
map evaluations until max|G(x_k) - x_k| < tol, and the error is against the fixed point."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
from paper_2307_12119_b200 import inputs

cfgname = sys.argv[1] if len(sys.argv) > 1 else "cfg1"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 6
law = int(sys.argv[3]) if len(sys.argv) > 3 else 0
scale = float(sys.argv[4]) if len(sys.argv) > 4 else 1.0
g = np.load(Path(__file__).resolve().parents[1] / "tests/golden/greens_n256.npz")
n = 256
m, c = 2 * n, n // 2
K = np.zeros((m, m))
x = (np.arange(n) - c) % m
K[np.ix_(x, x)] = g["f_sp0"] - float(g["phi"])
fk = np.fft.rfft2(K)
fk[0, 0] += float(g["phi"]) * m * m / 4
beta, leak_frac, tol = 0.017, 0.3, 1e-4
cfg = inputs.CONFIGS[cfgname]
P, V = inputs.mc_inputs(cfg, 0, B)
P = np.asarray(P, dtype=np.float64) * scale
V = np.asarray(V, dtype=np.float64)


def make_G(p, v):
    L0 = leak_frac * p * v

    def G(T):
        app = p + L0 * ((1 + beta * T) if law == 0 else np.exp(beta * T))
        mir = np.concatenate([app, app[::-1]], 0)
        mir = np.concatenate([mir, mir[:, ::-1]], 1)
        return np.fft.irfft2(fk * np.fft.rfft2(mir), s=(m, m))[:n, :n]
    return G


def picard(G, tol, maxit=400):
    T = np.zeros((n, n))
    for it in range(1, maxit + 1):
        Tn = G(T)
        d = np.abs(Tn - T).max()
        T = Tn
        if it > 1 and d < tol:
            return T, it
    return T, maxit


def cheb(G, k0, tol, maxit=200):
    xm = None
    x = np.zeros((n, n))
    res_prev = 0.0
    omega = 0.0
    for it in range(1, maxit + 1):
        gx = G(x)
        res = np.abs(gx - x).max()
        if it > 1 and res < tol:
            return gx, it
        if omega > 0:
            omega = 2 / (2 - s2) if omega == 1.0 else 1 / (1 - 0.25 * s2 * omega)
        elif it == k0 and res_prev > 0:
            rho = min(0.97, 1.02 * res / res_prev)
            gamma = 2 / (2 - rho)
            s2 = (rho / (2 - rho)) ** 2
            omega = 1.0
        res_prev = res
        if omega > 0:
            xn = omega * (gamma * gx + (1 - gamma) * x - xm) + xm if omega != 1.0 else gamma * gx + (1 - gamma) * x
        else:
            xn = gx
        xm, x = x, xn
    return x, maxit


def anderson(G, mdepth, tol, maxit=200, start=1):
    x = np.zeros((n, n))
    dX, dF = [], []
    xo = fo = None
    for it in range(1, maxit + 1):
        gx = G(x)
        f = gx - x
        res = np.abs(f).max()
        if it > 1 and res < tol:
            return gx, it
        if xo is not None:
            dX.append((gx - go).ravel())   # differences of G values
            dF.append((f - fo).ravel())
            dX, dF = dX[-mdepth:], dF[-mdepth:]
        go, fo = gx, f
        if it > start and dF:
            A = np.stack(dF, 1)
            gam = np.linalg.lstsq(A, f.ravel(), rcond=None)[0]
            xn = gx - (np.stack(dX, 1) @ gam).reshape(n, n)
        else:
            xn = gx
        xo, x = x, xn
    return x, maxit


rows = []
for b in range(B):
    G = make_G(P[b], V[b])
    Tstar, itp = picard(G, 1e-11)
    _, it_pic = picard(G, tol)
    out = {"picard": it_pic}
    for k0 in (3, 5):
        T, it = cheb(G, k0, tol)
        out[f"cheb{k0}"] = (it, float(np.abs(T - Tstar).max()))
    for md in (1, 2, 3, 5):
        T, it = anderson(G, md, tol)
        out[f"aa{md}"] = (it, float(np.abs(T - Tstar).max()))
    print(b, f"peak {Tstar.max():.1f} K", out, flush=True)


def deflated(G, p, v, tol, variant, maxit=200, cheb_k0=0):
    """x_{k+1} = g_k + delta_k (uniform shift): rank-one coarse correction of the constant mode."""
    L0 = leak_frac * p * v
    W = L0.sum()
    # h = G[L0 v] - the response to the nominal leakage alone (linear law: G is affine, take the difference)
    zero = np.zeros((n, n))
    app = L0
    mir = np.concatenate([app, app[::-1]], 0)
    mir = np.concatenate([mir, mir[:, ::-1]], 1)
    h = np.fft.irfft2(fk * np.fft.rfft2(mir), s=(m, m))[:n, :n]
    phi = float(g["phi"])
    x = zero
    evals = 1  # h costs one evaluation
    for it in range(1, maxit + 1):
        gx = G(x)
        evals += 1
        f = gx - x
        res = np.abs(f).max()
        if it > 1 and res < tol:
            return gx, evals
        if variant == 1:
            delta = beta * phi * (L0 * f).sum() / (1 - beta * phi * W)
        else:
            delta = beta * (L0 * h * f).sum() / (W - beta * (L0 * h).sum())
        x = gx + delta
    return x, maxit


for b in range(B):
    G = make_G(P[b], V[b])
    Tstar, _ = picard(G, 1e-11)
    out = {}
    for var in (1, 2):
        T, ev = deflated(G, P[b], V[b], tol, var)
        out[f"defl{var}"] = (ev, float(np.abs(T - Tstar).max()))
    print(b, out, flush=True)
