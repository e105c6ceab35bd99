"""Seeded synthetic observation generator (numpy PCG64).

Recipe: `default_rng(cfg.gen_seed)` draws, in
this order, bump centres (uniform in the domain), amplitudes U(-1, 1), widths
(uniform or log-uniform), observation positions, observation noise.

The field f stands in for the paper's missing Tangle / ethanediol SGPR models
(PAPER.md:310-328): a sum of isotropic Gaussian bumps a*exp(-|x-c|^2/(2w^2))
plus optional linear ramp / sin texture, or the c1 analytic field
sin(2 pi x) cos(2 pi y) + 0.5 z.  Observations y = f(x) + N(0, noise_std^2).

Placement "grad" draws positions by rejection with density proportional to
|grad f| (envelope 1.25 x the maximum over a 64^3 probe lattice); "mixed" draws
the first half uniformly and the second half by gradient.
"""
from __future__ import annotations

import dataclasses
import functools
from typing import List

import numpy as np

from .configs import Config, get_config


@dataclasses.dataclass
class Field:
    cfg: Config
    centres: np.ndarray
    amps: np.ndarray
    widths: np.ndarray

    def value(self, x: np.ndarray) -> np.ndarray:
        cfg = self.cfg
        x = np.asarray(x, dtype=np.float64)
        out = np.zeros(x.shape[0])
        if cfg.tangle_like:
            out += np.sin(2 * np.pi * x[:, 0]) * np.cos(2 * np.pi * x[:, 1]) + 0.5 * x[:, 2]
        for s in range(0, x.shape[0], 65536):
            xs = x[s:s + 65536]
            if len(self.amps):
                d2 = ((xs[:, None, :] - self.centres[None, :, :]) ** 2).sum(-1)
                out[s:s + 65536] += (self.amps[None, :] *
                                     np.exp(-d2 / (2 * self.widths[None, :] ** 2))).sum(-1)
        out += cfg.ramp_z * x[:, 2]
        out += cfg.texture_sin4pix * np.sin(4 * np.pi * x[:, 0])
        return out

    def grad_norm(self, x: np.ndarray) -> np.ndarray:
        cfg = self.cfg
        g = np.zeros_like(x)
        if cfg.tangle_like:
            g[:, 0] += 2 * np.pi * np.cos(2 * np.pi * x[:, 0]) * np.cos(2 * np.pi * x[:, 1])
            g[:, 1] += -2 * np.pi * np.sin(2 * np.pi * x[:, 0]) * np.sin(2 * np.pi * x[:, 1])
            g[:, 2] += 0.5
        for s in range(0, x.shape[0], 16384):
            xs = x[s:s + 16384]
            if len(self.amps):
                diff = xs[:, None, :] - self.centres[None, :, :]
                d2 = (diff ** 2).sum(-1)
                w2 = self.widths[None, :] ** 2
                e = self.amps[None, :] * np.exp(-d2 / (2 * w2))
                g[s:s + 16384] += (-(e / w2)[:, :, None] * diff).sum(1)
        g[:, 2] += cfg.ramp_z
        g[:, 0] += cfg.texture_sin4pix * 4 * np.pi * np.cos(4 * np.pi * x[:, 0])
        return np.sqrt((g ** 2).sum(-1))


@dataclasses.dataclass
class Workload:
    cfg: Config
    X: np.ndarray          # (m, 3) float64, row-major
    y: np.ndarray          # (m,) float64
    thetas: List[float]    # resolved isovalues
    field: Field


def _uniform(rng, cfg, n):
    lo = np.asarray(cfg.lo)
    hi = np.asarray(cfg.hi)
    return lo + (hi - lo) * rng.random((n, 3))


def _by_gradient(rng, cfg, field, n):
    lo = np.asarray(cfg.lo)
    hi = np.asarray(cfg.hi)
    t = (np.arange(64) + 0.5) / 64.0
    probe = np.stack(np.meshgrid(t, t, t, indexing="ij"), -1).reshape(-1, 3)
    env = 1.25 * field.grad_norm(lo + (hi - lo) * probe).max()
    out = []
    have = 0
    while have < n:
        cand = _uniform(rng, cfg, 4 * n)
        acc = rng.random(4 * n) * env < field.grad_norm(cand)
        cand = cand[acc]
        out.append(cand)
        have += len(cand)
    return np.concatenate(out)[:n]


@functools.lru_cache(maxsize=16)
def generate(name: str) -> Workload:
    cfg = get_config(name)
    rng = np.random.default_rng(cfg.gen_seed)
    lo = np.asarray(cfg.lo)
    hi = np.asarray(cfg.hi)
    nb = cfg.n_bumps
    centres = lo + (hi - lo) * rng.random((nb, 3))
    amps = rng.uniform(-1.0, 1.0, nb)
    if cfg.width_log:
        widths = np.exp(rng.uniform(np.log(cfg.width_lo), np.log(cfg.width_hi), nb))
    else:
        widths = rng.uniform(cfg.width_lo, cfg.width_hi, nb)
    field = Field(cfg, centres, amps, widths)
    if cfg.placement == "uniform":
        X = _uniform(rng, cfg, cfg.m)
    elif cfg.placement == "grad":
        X = _by_gradient(rng, cfg, field, cfg.m)
    elif cfg.placement == "mixed":
        h = cfg.m // 2
        X = np.concatenate([_uniform(rng, cfg, h), _by_gradient(rng, cfg, field, cfg.m - h)])
    else:
        raise ValueError(cfg.placement)
    y = field.value(X) + cfg.noise_std * rng.standard_normal(cfg.m)
    thetas = []
    for th in cfg.thetas:
        if th is None:
            # median of the noise-free field over the vertex lattice (reading R22)
            axes = [lo[d] + np.arange(cfg.cells[d] + 1) * ((hi[d] - lo[d]) / cfg.cells[d])
                    for d in range(3)]
            V = np.stack(np.meshgrid(*axes, indexing="ij"), -1).reshape(-1, 3)
            th = float(np.median(field.value(V)))
        thetas.append(float(th))
    X = np.ascontiguousarray(X, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    X.setflags(write=False)
    y.setflags(write=False)
    return Workload(cfg, X, y, thetas, field)


def random_cells(name: str, n: int, seed: int) -> np.ndarray:
    """Seeded sample of distinct linear cell ids (x fastest) of a config's grid."""
    cfg = get_config(name)
    total = cfg.cells[0] * cfg.cells[1] * cfg.cells[2]
    rng = np.random.default_rng(seed)
    n = min(n, total)
    return np.sort(rng.choice(total, size=n, replace=False)).astype(np.int64)


def morton_sorted_cells(cells, c0=0, c1=None, device=None):
    """Linear cell ids [c0, c1) of a grid (x fastest) in Morton order of (i, j, k), as an int64
    torch tensor: the input order under which a dense cell list takes the 4^3-brick posterior
    kernels (a list ordering, not part of the method)."""
    import torch
    nx, ny, nz = cells
    if c1 is None:
        c1 = nx * ny * nz
    c = torch.arange(c0, c1, dtype=torch.int64, device=device)

    def spread(v):
        out = torch.zeros_like(v)
        for bit in range(21):
            out |= ((v >> bit) & 1) << (3 * bit)
        return out

    key = spread(c % nx) | (spread((c // nx) % ny) << 1) | (spread(c // (nx * ny)) << 2)
    return c[torch.argsort(key)]
