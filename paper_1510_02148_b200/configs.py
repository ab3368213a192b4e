"""Seeded synthetic inputs with the shapes of BASELINE.json's five configurations.

Every generator is deterministic in (config, seed) and returns host arrays (k fields, the
DIA operator, b and the partition), so the device path and the CPU oracle consume identical
inputs.  Common settings: mu = 1, unscaled A, right Jacobi, A_p = A,
x0 = 0, tol = 1e-8, Dirichlet faces through the ghost half-cell rule with boundary_perm 1.

Config 3 is a synthetic stand-in with the shape of the public SPE10-model-2-like case the
paper uses; no dataset values are used or reproduced.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .testbed import BoundarySpec, Grid, PermeabilityField, assemble_dia
from .sparse import SparseMatrix


@dataclass
class Case:
    name: str
    grid: Grid
    field: PermeabilityField
    band_field: PermeabilityField   # field whose kx drives the levelset banding
    bc: BoundarySpec
    boxes: tuple
    jump_threshold: float
    m: int
    tol: float = 1e-8
    max_iters: int = 20000
    seed: int = 0

    def problem(self):
        """(A as SparseMatrix, b)."""
        off, dg, b = assemble_dia(self.field, self.bc)
        return SparseMatrix.from_dia(self.grid.n_cells, off, dg), b

    def partition(self):
        from .physics import subdomain_levelset_partition
        px, py, pz = self.boxes
        return subdomain_levelset_partition(self.band_field, px, py, pz, self.jump_threshold)


X_FACES = BoundarySpec(top_dirichlet=False, faces=(("xmin", 1.0), ("xmax", 0.0)))
Y_FACES = BoundarySpec(top_dirichlet=False, faces=(("ymin", 1.0), ("ymax", 0.0)))


def _layered(grid: Grid, per_z_kx: np.ndarray, kz_factor: float = 1.0) -> PermeabilityField:
    kx = np.repeat(np.asarray(per_z_kx, dtype=np.float64), grid.nx * grid.ny)
    return PermeabilityField(grid, kx, kx.copy(), kx * kz_factor)


def config1(seed: int = 0) -> Case:
    """32^3, 4 z-blocks alternating k = 1, 1e-4; x-face Dirichlet; 2x2x2 boxes; d = 16."""
    g = Grid(32, 32, 32)
    per_z = np.repeat([1.0, 1e-4, 1.0, 1e-4], 8)
    f = _layered(g, per_z)
    return Case("32x32x32", g, f, f, X_FACES, (2, 2, 2), 2.0, m=50, seed=seed)


def config2(seed: int = 0) -> Case:
    """128x128x64, 8 layers of 8 cells, k per layer from {1,1e-2,1e-4,1e-6}, kz = 0.1 kx."""
    rng = np.random.default_rng(seed)
    g = Grid(128, 128, 64)
    per_layer = rng.choice(np.array([1.0, 1e-2, 1e-4, 1e-6]), size=8)
    per_z = np.repeat(per_layer, 8)
    f = _layered(g, per_z, 0.1)
    return Case("128x128x64", g, f, f, X_FACES, (4, 4, 4), 1.0, m=50, seed=seed)


def _box_filter(a: np.ndarray, w: int, axes) -> np.ndarray:
    """Mean over a centred window of w cells along each axis in `axes` (edge-clamped)."""
    out = a
    for ax in axes:
        pad = [(0, 0)] * out.ndim
        pad[ax] = (w // 2, w - 1 - w // 2)
        p = np.pad(out, pad, mode="edge")
        c = np.cumsum(p, axis=ax)
        zero = np.zeros_like(np.take(c, [0], axis=ax))
        c = np.concatenate([zero, c], axis=ax)
        n = out.shape[ax]
        hi = np.take(c, np.arange(w, w + n), axis=ax)
        lo = np.take(c, np.arange(0, n), axis=ax)
        out = (hi - lo) / w
    return out


def config3(seed: int = 0) -> Case:
    """60x220x85 two-zone heterogeneous case, cells 20x10x2 ft (BASELINE configs[2]).

    Top 35 layers (iz >= 50, the reference's 'top' is the highest iz): log10 kx ~ N(0, 1)
    per cell, correlated by a 3D 5-cell box filter, renormalised to unit standard deviation
    (the box filter alone shrinks it to ~0.09), clipped to [-3, 3].
    Bottom 50 layers: kx = 1e-3 with 6 sinusoidal channels per layer at 1e3; each channel
    runs along y, 4-8 cells wide in x, amplitude 5-20 cells, wavelength 60-160 cells, random
    centre and phase.  ky = kx, kz = 0.1 kx.  Dirichlet p = 1 on y = 0, p = 0 on y = 219.
    Banding: 4 bins of log10 k with edges -1.5, 0, 1.5, expressed through the unchanged
    partition API as a banding field kx = 10**(2*bin) with jump_threshold = 1.0.
    """
    rng = np.random.default_rng(seed)
    g = Grid(60, 220, 85, 20.0, 10.0, 2.0)
    nz_top, nz_bot = 35, 50
    logk = np.empty((g.nz, g.ny, g.nx))
    z = rng.standard_normal((nz_top, g.ny, g.nx))
    z = _box_filter(z, 5, axes=(0, 1, 2))
    z = (z - z.mean()) / z.std()
    logk[nz_bot:] = np.clip(z, -3.0, 3.0)
    bot = np.full((nz_bot, g.ny, g.nx), -3.0)
    iy = np.arange(g.ny)[:, None]
    ix = np.arange(g.nx)[None, :]
    for iz in range(nz_bot):
        for _ in range(6):
            width = rng.integers(4, 9)
            amp = rng.uniform(5.0, 20.0)
            lam = rng.uniform(60.0, 160.0)
            phase = rng.uniform(0.0, 2.0 * np.pi)
            x0 = rng.uniform(0.0, g.nx)
            xc = x0 + amp * np.sin(2.0 * np.pi * iy / lam + phase)
            bot[iz][np.abs(ix - xc) < width / 2.0] = 3.0
    logk[:nz_bot] = bot
    kx = 10.0 ** logk.ravel()
    f = PermeabilityField(g, kx, kx.copy(), 0.1 * kx)
    bins = np.searchsorted(np.array([-1.5, 0.0, 1.5]), logk.ravel(), side="right")
    kb = 10.0 ** (2.0 * bins)
    fb = PermeabilityField(g, kb, kb.copy(), kb.copy())
    return Case("60x220x85", g, f, fb, Y_FACES, (6, 11, 5), 1.0, m=50, seed=seed)


def config4(seed: int = 0) -> Case:
    """256^3, 16 layers of seeded thickness 4-32 summing to 256, log10 k random walk."""
    rng = np.random.default_rng(seed)
    g = Grid(256, 256, 256)
    while True:
        t = rng.integers(4, 33, size=16)
        if t.sum() == 256:
            break
    logs = [0.0]
    for _ in range(15):
        logs.append(logs[-1] + rng.choice([-1.0, 1.0]) * rng.uniform(4.0, 6.0))
    per_z = np.repeat(10.0 ** np.array(logs), t)
    f = _layered(g, per_z)
    return Case("256x256x256", g, f, f, X_FACES, (8, 8, 8), 2.0, m=50, seed=seed)


def config5(seed: int = 0) -> Case:
    """512x512x256, k = 1 with 4000 cuboids (edges 4-24) at 1e-6; 16x16x8 boxes; m = 40."""
    rng = np.random.default_rng(seed)
    g = Grid(512, 512, 256)
    k = np.ones((g.nz, g.ny, g.nx))
    for _ in range(4000):
        ex, ey, ez = rng.integers(4, 25, size=3)
        x0 = rng.integers(0, g.nx - ex + 1)
        y0 = rng.integers(0, g.ny - ey + 1)
        z0 = rng.integers(0, g.nz - ez + 1)
        k[z0:z0 + ez, y0:y0 + ey, x0:x0 + ex] = 1e-6
    kx = k.ravel()
    f = PermeabilityField(g, kx, kx.copy(), kx.copy())
    return Case("512x512x256", g, f, f, X_FACES, (16, 16, 8), 2.0, m=40, seed=seed)


CONFIGS = {1: config1, 2: config2, 3: config3, 4: config4, 5: config5}


def make_case(index: int, seed: int = 0) -> Case:
    return CONFIGS[index](seed)
