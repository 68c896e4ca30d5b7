"""Seeded synthetic stand-ins for the five BASELINE.json configs.

The paper's canonical test images are not available, so every
config is a seeded generator with the shapes and value distributions
BASELINE.json states. Image seeds: cfg s uses seed s
(s = 1..4); cfg5 image i uses seed 1000 + i. WSM init seed = 1 (the CLI
default, tools/colorq.cpp:73); termination = convergent(1e-4, cap 100).

All generators use numpy's PCG64 (bit-stable across platforms), produce
row-major ``uint8[H, W, 3]`` rasters (the reference's RgbImage layout,
color.hpp:57-75) and round with ``lround`` semantics (half away from zero,
then clamp; color.hpp:38-46).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def round_to_u8(x: np.ndarray) -> np.ndarray:
    """color.hpp:38-46 — lround (half away from zero) then clamp to [0, 255]."""
    r = np.where(x >= 0, np.floor(x + 0.5), np.ceil(x - 0.5))
    return np.clip(r, 0, 255).astype(np.uint8)


def gmm_image(width: int, height: int, components: int, seed: int) -> np.ndarray:
    """Pixels iid from an isotropic Gaussian mixture in RGB: means U[0,255]^3,
    sigma U[4,20], mixture weights Dirichlet(1) (configs 1, 2, 5)."""
    rng = np.random.default_rng(seed)
    means = rng.uniform(0.0, 255.0, size=(components, 3))
    sigma = rng.uniform(4.0, 20.0, size=components)
    weights = rng.dirichlet(np.ones(components))
    p = width * height
    comp = rng.choice(components, size=p, p=weights)
    x = means[comp] + sigma[comp, None] * rng.standard_normal(size=(p, 3))
    return round_to_u8(x).reshape(height, width, 3)


def value_noise_image(width: int, height: int, seed: int, cells=(512, 128, 32, 8),
                      amps=(128.0, 64.0, 32.0, 16.0), noise_sigma: float = 8.0) -> np.ndarray:
    """Photo-like: per channel, sum of 4 octaves of bilinear value noise over a
    U[0,1] lattice (cell sizes 512/128/32/8 px, amplitudes 128/64/32/16) plus
    iid N(0, 8), rounded and clipped (config 3; SURVEY.md §8(d) lattice note)."""
    rng = np.random.default_rng(seed)
    out = np.zeros((height, width, 3), np.float64)
    ys = np.arange(height, dtype=np.float64)
    xs = np.arange(width, dtype=np.float64)
    for ch in range(3):
        acc = np.zeros((height, width), np.float64)
        for cell, amp in zip(cells, amps):
            gy = height // cell + 2
            gx = width // cell + 2
            lat = rng.uniform(0.0, 1.0, size=(gy, gx))
            fy = ys / cell
            fx = xs / cell
            iy = np.floor(fy).astype(np.int64)
            ix = np.floor(fx).astype(np.int64)
            ty = (fy - iy)[:, None]
            tx = (fx - ix)[None, :]
            v00 = lat[iy][:, ix]
            v01 = lat[iy][:, ix + 1]
            v10 = lat[iy + 1][:, ix]
            v11 = lat[iy + 1][:, ix + 1]
            top = v00 + (v01 - v00) * tx
            bot = v10 + (v11 - v10) * tx
            acc += amp * (top + (bot - top) * ty)
        out[..., ch] = acc
    out += noise_sigma * rng.standard_normal(size=out.shape)
    return round_to_u8(out)


def uniform_image(width: int, height: int, seed: int) -> np.ndarray:
    """iid uniform 24-bit pixels (config 4, worst-case data reduction)."""
    rng = np.random.default_rng(seed)
    keys = rng.integers(0, 1 << 24, size=width * height, dtype=np.uint32)
    img = np.empty((width * height, 3), np.uint8)
    img[:, 0] = (keys >> 16) & 255
    img[:, 1] = (keys >> 8) & 255
    img[:, 2] = keys & 255
    return img.reshape(height, width, 3)


@dataclass(frozen=True)
class Config:
    name: str
    width: int
    height: int
    ks: tuple
    description: str
    images: int = 1

    @property
    def pixels(self) -> int:
        return self.width * self.height

    def image(self, index: int = 0, seed: int | None = None) -> np.ndarray:
        if self.name == "cfg1":
            return gmm_image(self.width, self.height, 64, 1 if seed is None else seed)
        if self.name == "cfg2":
            return gmm_image(self.width, self.height, 256, 2 if seed is None else seed)
        if self.name == "cfg3":
            return value_noise_image(self.width, self.height, 3 if seed is None else seed)
        if self.name == "cfg4":
            return uniform_image(self.width, self.height, 4 if seed is None else seed)
        if self.name == "cfg5":
            return gmm_image(self.width, self.height, 256, 1000 + index if seed is None else seed)
        raise KeyError(self.name)


CONFIGS = {
    "cfg1": Config("cfg1", 512, 512, (32,), "GMM-64"),
    "cfg2": Config("cfg2", 768, 512, (64, 256), "GMM-256"),
    "cfg3": Config("cfg3", 4096, 4096, (256,), "4-octave value noise + N(0,8)"),
    "cfg4": Config("cfg4", 4096, 4096, (256,), "uniform 24-bit"),
    "cfg5": Config("cfg5", 1024, 1024, (64, 256), "64 GMM-256 images", images=64),
}

# BASELINE.json termination: relative SSE change <= 1e-4 or 100 iterations.
EPSILON = 1e-4
HARD_CAP = 100
INIT_SEED = 1
