"""Seeded synthetic inputs for the BASELINE.json configs.

BASELINE names no public benchmark or dataset; these generators stand in for
the paper's floorplans with the shapes, sizes and value distributions the
configs state:
  * power maps: seeded guillotine floorplan (split the largest block along its
    longer side at U[0.3, 0.7], snapped to cells) with per-block density
    U[0.2, 2.0] W/mm^2, plus optional Gaussian hotspots (sigma 0.5 mm, peak
    U[5, 10] W/mm^2) added on top;
  * variation maps: var = 1 + (sigma/mu) * z, z a unit-variance Gaussian random
    field with the reference's spherical correlogram (variation.cpp:75-79) made
    by circulant embedding on the 2n torus (the construction of
    gen_systematic_map, variation.cpp:87-132, with torch's RNG);
  * Markov power traces for the transient config.
Every sample i has its own seed derived as in the reference's derived_seed
(splitmix64, variation.cpp:68-85), so a sample does not depend on the batch
size or on how samples are sharded over GPUs.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

MASK64 = (1 << 64) - 1


def splitmix64(x: int) -> int:
    x = (x + 0x9E3779B97F4A7C15) & MASK64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & MASK64
    return x ^ (x >> 31)


def sample_seed(base: int, purpose: int, run: int) -> int:
    return splitmix64((base ^ (purpose << 32) ^ (run * 0x51ED2701)) & MASK64)


PURPOSE_POWER, PURPOSE_VAR, PURPOSE_TRACE = 0x41, 0x42, 0x43


@dataclass(frozen=True)
class Config:
    name: str
    n: int
    die_mm: float
    blocks: int
    hotspots: int
    sigma_over_mu: float
    corr_range: float
    batch: int
    base_seed: int

    @property
    def pitch_mm(self) -> float:
        return self.die_mm / self.n


CONFIGS = {
    "cfg0": Config("cfg0", 64, 16.0, 16, 0, 0.10, 0.5, 1, 1),
    "cfg1": Config("cfg1", 256, 16.0, 32, 4, 0.10, 0.5, 4096, 1001),
    "cfg2": Config("cfg2", 1024, 16.0, 32, 4, 0.15, 0.25, 256, 2001),
    "cfg3": Config("cfg3", 512, 16.0, 32, 0, 0.10, 0.5, 64, 3001),
    "cfg4": Config("cfg4", 8192, 16.0, 1024, 64, 0.10, 0.5, 1, 4001),
}


def guillotine_blocks(n: int, leaves: int, rng: np.random.Generator) -> list[tuple[int, int, int, int]]:
    blocks = [(0, n, 0, n)]
    while len(blocks) < leaves:
        areas = [(b[1] - b[0]) * (b[3] - b[2]) for b in blocks]
        k = int(np.argmax(areas))
        r0, r1, c0, c1 = blocks[k]
        h, w = r1 - r0, c1 - c0
        if max(h, w) < 2:
            break
        frac = rng.uniform(0.3, 0.7)
        blocks.pop(k)
        if h >= w:
            s = r0 + min(max(int(round(h * frac)), 1), h - 1)
            blocks += [(r0, s, c0, c1), (s, r1, c0, c1)]
        else:
            s = c0 + min(max(int(round(w * frac)), 1), w - 1)
            blocks += [(r0, r1, c0, s), (r0, r1, s, c1)]
    return blocks


def power_map(cfg: Config, index: int) -> np.ndarray:
    """Watts per cell, float64 (n, n)."""
    rng = np.random.default_rng(sample_seed(cfg.base_seed, PURPOSE_POWER, index))
    n, pm = cfg.n, cfg.pitch_mm
    dens = np.zeros((n, n))
    for r0, r1, c0, c1 in guillotine_blocks(n, cfg.blocks, rng):
        dens[r0:r1, c0:c1] = rng.uniform(0.2, 2.0)
    if cfg.hotspots:
        x = (np.arange(n) + 0.5) * pm
        for _ in range(cfg.hotspots):
            cx, cy = rng.uniform(0.0, cfg.die_mm, size=2)
            peak = rng.uniform(5.0, 10.0)
            gx = np.exp(-((x - cx) ** 2) / (2 * 0.5 ** 2))
            gy = np.exp(-((x - cy) ** 2) / (2 * 0.5 ** 2))
            dens += peak * np.outer(gx, gy)
    return dens * pm * pm


def power_map_torch(cfg: Config, index: int, device="cuda"):
    """power_map for large grids (config 4): identical draws, the hotspot sum and the
    block fill done with torch on `device` (float64 (n, n) tensor, W per cell)."""
    import torch
    rng = np.random.default_rng(sample_seed(cfg.base_seed, PURPOSE_POWER, index))
    n, pm = cfg.n, cfg.pitch_mm
    dens = torch.zeros((n, n), dtype=torch.float64, device=device)
    for r0, r1, c0, c1 in guillotine_blocks(n, cfg.blocks, rng):
        dens[r0:r1, c0:c1] = rng.uniform(0.2, 2.0)
    if cfg.hotspots:
        x = (torch.arange(n, dtype=torch.float64, device=device) + 0.5) * pm
        for _ in range(cfg.hotspots):
            cx, cy = rng.uniform(0.0, cfg.die_mm, size=2)
            peak = rng.uniform(5.0, 10.0)
            gx = torch.exp(-((x - cx) ** 2) / (2 * 0.5 ** 2))
            gy = torch.exp(-((x - cy) ** 2) / (2 * 0.5 ** 2))
            dens += peak * torch.outer(gx, gy)
    return dens * pm * pm


def power_batch(cfg: Config, start: int, count: int, dtype=np.float32) -> np.ndarray:
    out = np.empty((count, cfg.n, cfg.n), dtype=dtype)
    for k in range(count):
        out[k] = power_map(cfg, start + k)
    return out


def spherical_eigs(n: int, pitch_mm: float, range_mm: float) -> np.ndarray:
    """Circulant-embedding eigenvalues of the spherical correlogram on the
    2n torus, clamped >= 0 and rescaled to unit marginal variance."""
    m = 2 * n
    d1 = np.minimum(np.arange(m), m - np.arange(m)) * pitch_mm
    d = np.hypot(d1[:, None], d1[None, :])
    x = d / range_mm
    cov = np.where(d < range_mm, 1.0 - 1.5 * x + 0.5 * x ** 3, 0.0)
    lam = np.maximum(np.fft.fft2(cov).real, 0.0)
    return lam * (m * m / lam.sum())


def variation_batch(cfg: Config, start: int, count: int, device: str = "cpu", dtype=None, chunk: int = 64):
    """torch tensor (count, n, n): var = 1 + (sigma/mu) z."""
    import torch
    dtype = dtype or torch.float32
    n, m = cfg.n, 2 * cfg.n
    sq = torch.from_numpy(np.sqrt(spherical_eigs(n, cfg.pitch_mm, cfg.corr_range * cfg.die_mm))).to(device)
    out = torch.empty((count, n, n), dtype=dtype, device=device)
    for c0 in range(0, count, chunk):
        cc = min(chunk, count - c0)
        noise = torch.empty((cc, m, m), dtype=torch.float64, device=device)
        for k in range(cc):
            g = torch.Generator(device=device)
            g.manual_seed(sample_seed(cfg.base_seed, PURPOSE_VAR, start + c0 + k) & ((1 << 63) - 1))
            noise[k] = torch.randn((m, m), generator=g, dtype=torch.float64, device=device)
        z = torch.fft.ifft2(torch.fft.fft2(noise) * sq).real[:, :n, :n]
        out[c0:c0 + cc] = (1.0 + cfg.sigma_over_mu * z).to(dtype)
    return out


def mc_inputs(cfg: Config, start: int, count: int, device: str = "cpu", torch_dtype=None):
    """(p_dyn, var) torch tensors of one shard of a config's MC batch."""
    import torch
    torch_dtype = torch_dtype or torch.float32
    np_dt = np.float64 if torch_dtype == torch.float64 else np.float32
    p = torch.from_numpy(power_batch(cfg, start, count, np_dt)).to(device)
    v = variation_batch(cfg, start, count, device=device, dtype=torch_dtype)
    return p, v


def markov_blocks(cfg: Config, index: int, steps: int, switch_prob: float = 1.0 / 50.0,
                  off_frac: float = 0.1):
    """Compact form of trace `index`: per-block two-state Markov chain (on
    density U[0.5, 2] W/mm^2 drawn once per block, off at off_frac of it,
    switching with probability switch_prob per step = mean dwell 50 steps).
    Returns (blk (n, n) int32 block ids, sched (steps, nblk) W/cell per block and
    step, on (n, n) W/cell of the all-on state)."""
    rng = np.random.default_rng(sample_seed(cfg.base_seed, PURPOSE_TRACE, index))
    n, pm = cfg.n, cfg.pitch_mm
    blocks = guillotine_blocks(n, cfg.blocks, rng)
    on = rng.uniform(0.5, 2.0, size=len(blocks))
    state = rng.random(len(blocks)) < 0.5
    blk = np.zeros((n, n), np.int32)
    on_map = np.zeros((n, n))
    for b, (r0, r1, c0, c1) in enumerate(blocks):
        blk[r0:r1, c0:c1] = b
        on_map[r0:r1, c0:c1] = on[b] * pm * pm
    sched = np.empty((steps, len(blocks)))
    for t in range(steps):
        flip = rng.random(len(blocks)) < switch_prob
        state = np.where(flip, ~state, state)
        sched[t] = on * np.where(state, 1.0, off_frac) * pm * pm
    return blk, sched, on_map


def markov_trace(cfg: Config, index: int, steps: int, switch_prob: float = 1.0 / 50.0,
                 off_frac: float = 0.1) -> np.ndarray:
    """(steps, n, n) W/cell frames of trace `index` (markov_blocks expanded)."""
    blk, sched, _ = markov_blocks(cfg, index, steps, switch_prob, off_frac)
    return sched[:, blk]
