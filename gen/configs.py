"""The five synthetic workloads of BASELINE.json (`configs[0..4]`), C1..C5.

Recipes are SURVEY.md §8(d) with the readings listed in DESIGN.md §Readings
(spectrum indexing = reading R9, unscaled Gaussian entries = R10, C3 clamp =
R7, CT geometry = R12/R13, X and T for C3..C5 = R14).  This file only states
sizes, seeds and the spectrum recipe; it computes nothing of the method.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


def spectrum(W: int):
    """BASELINE.json configs[0]: s_j ∝ exp(-(j - W/2)^2 / (2 (W/4)^2)), 0-based j
    (reading R9), normalised in fp64; mu_j = linspace(2.0, 0.5, W)."""
    j = np.arange(W, dtype=np.float64)
    s = np.exp(-((j - W / 2.0) ** 2) / (2.0 * (W / 4.0) ** 2))
    s = s / s.sum()
    mu = np.linspace(2.0, 0.5, W) if W > 1 else np.array([1.0])
    return s, mu


SET_NONE, SET_BALL, SET_NONNEG, SET_NONNEG_BALL = 0, 1, 2, 3


@dataclass(frozen=True)
class Config:
    name: str
    n: int
    d: int
    W: int
    I_bar: float
    seed: int
    T: int
    radius: float            # X = B(radius) (ball set) or its radius part
    set: int = SET_BALL
    dtype: str = "f32"       # element type of A
    kind: str = "dense"      # dense | reparam | csr
    x_star_radius: float = 1.0
    sigma: float = 0.0       # electronic noise (C4)
    extra: dict = field(default_factory=dict)

    @property
    def spectrum(self):
        return spectrum(self.W)


C1 = Config("c1", n=2000, d=100, W=10, I_bar=1e4, seed=0, T=100, radius=1.0, dtype="f64")
C1F = Config("c1f32", n=2000, d=100, W=10, I_bar=1e4, seed=0, T=100, radius=1.0, dtype="f32")
C2 = Config("c2", n=200_000, d=1024, W=20, I_bar=1e4, seed=1, T=200, radius=1.0)
C3 = Config("c3", n=1_000_000, d=512, W=16, I_bar=5e4, seed=2, T=100, radius=0.5,
            kind="reparam", x_star_radius=0.5)
C4 = Config("c4", n=360 * 367, d=256 * 256, W=16, I_bar=1e5, seed=3, T=100, radius=0.0,
            set=SET_NONNEG_BALL, kind="csr", sigma=5.0,
            extra={"side": 256, "views": 360, "bins": 367, "ellipses": 10})
C5 = Config("c5", n=8_000_000, d=4096, W=32, I_bar=1e4, seed=4, T=20, radius=1.0)

CONFIGS = {c.name: c for c in (C1, C1F, C2, C3, C4, C5)}


def scaled(cfg: Config, n: int) -> Config:
    """Same recipe with fewer rows (rows are keyed by global index, so the
    first n rows of a scaled config are bit-identical to the full config)."""
    from dataclasses import replace
    return replace(cfg, n=n)
