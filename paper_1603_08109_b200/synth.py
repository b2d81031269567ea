"""Seeded synthetic inputs for the five BASELINE.json configurations.

The paper's test images and scikit-image's `camera` are not available, so
these generators stand in for them.  Choices the
BASELINE recipes leave open are fixed here:

* RNG: `numpy.random.default_rng(seed)`; draws in this order: sinusoid
  parameters (fy, fx, phase per component), then rectangles (top, left,
  height, width, value per rectangle), then the noise field.
* Rectangles: top-left uniform over the image, side lengths uniform integers in
  [16, 256] (inclusive), value uniform in [0, 255]; clipped at the border and
  painted in draw order (later rectangles overwrite earlier ones).
* Sinusoids: 30 sin(2 pi (fx x / width + fy y / height) + phase), fx, fy
  uniform in [1, 20] cycles/image, phase uniform in [0, 2 pi).
* Order: field, then rectangles, then additive N(0, sigma^2) noise, then clip
  to [0, 255].  Arithmetic in float64 up to 4096^2, float32 above (memory);
  the result is cast to the config dtype.

`CONFIGS` records shape, dtype, kernel and order parameters per config.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Config:
    name: str
    height: int
    width: int
    batch: int
    dtype: str
    kind: str
    sigma_s: float | None
    half_width: int | None
    sigma_r: float
    order: int | None        # explicit N (c0, c1)
    delta: float | None      # delta drives N (c2-c4)
    seed: int
    n_rects: int
    noise_sigma: float
    smooth_field: bool

    @property
    def pixels(self) -> int:
        return self.batch * self.height * self.width


CONFIGS = {
    "c0": Config("c0", 512, 512, 1, "float64", "gaussian", 3.0, None, 40.0, 15, None,
                 1603, 40, 10.0, False),
    "c1": Config("c1", 1024, 1024, 1, "float32", "box", None, 5, 50.0, 10, None,
                 1604, 40, 15.0, False),
    "c2": Config("c2", 4096, 4096, 1, "float32", "gaussian", 5.0, None, 30.0, None, 1.0,
                 1605, 200, 20.0, True),
    "c3": Config("c3", 2048, 2048, 64, "float32", "gaussian", 8.0, None, 20.0, None, 1.0,
                 2000, 200, 20.0, True),
    "c4": Config("c4", 16384, 16384, 1, "float32", "box", None, 20, 25.0, None, 1.0,
                 1607, 3000, 10.0, True),
}


def synth_image(height: int, width: int, *, seed: int, n_rects: int, noise_sigma: float,
                smooth_field: bool, dtype="float32") -> np.ndarray:
    rng = np.random.default_rng(seed)
    work = np.float64 if height * width <= 4096 * 4096 else np.float32
    if smooth_field:
        params = rng.uniform([1.0, 1.0, 0.0], [20.0, 20.0, 2.0 * math.pi], size=(8, 3))
        y = np.arange(height, dtype=np.float64) / height
        x = np.arange(width, dtype=np.float64) / width
        img = np.full((height, width), 128.0, dtype=work)
        for fy, fx, ph in params:
            # sin(a + b) = sin a cos b + cos a sin b  keeps the field an outer-product sum.
            ay = 2.0 * math.pi * fy * y + ph
            bx = 2.0 * math.pi * fx * x
            img += (30.0 * np.sin(ay)).astype(work)[:, None] * np.cos(bx).astype(work)[None, :]
            img += (30.0 * np.cos(ay)).astype(work)[:, None] * np.sin(bx).astype(work)[None, :]
    else:
        img = np.full((height, width), 128.0, dtype=work)
    rects = np.empty((n_rects, 5))
    rects[:, 0] = rng.integers(0, height, n_rects)
    rects[:, 1] = rng.integers(0, width, n_rects)
    rects[:, 2] = rng.integers(16, 257, n_rects)
    rects[:, 3] = rng.integers(16, 257, n_rects)
    rects[:, 4] = rng.uniform(0.0, 255.0, n_rects)
    for top, left, hh, ww, val in rects:
        img[int(top):int(top + hh), int(left):int(left + ww)] = val
    img += rng.standard_normal((height, width), dtype=work) * work(noise_sigma)
    np.clip(img, 0.0, 255.0, out=img)
    return img.astype(dtype, copy=False)


def config_image(cfg: Config | str, index: int = 0, *, height: int | None = None,
                 width: int | None = None) -> np.ndarray:
    """Image `index` of a config (batch member for c3); optional smaller shape for crops/tests."""
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    return synth_image(height or cfg.height, width or cfg.width, seed=cfg.seed + index,
                       n_rects=cfg.n_rects, noise_sigma=cfg.noise_sigma,
                       smooth_field=cfg.smooth_field, dtype=cfg.dtype)


def config_kernel(cfg: Config | str):
    from .kernels import make_spatial_kernel
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    if cfg.kind == "box":
        return make_spatial_kernel("box", half_width=cfg.half_width)
    return make_spatial_kernel("gaussian", sigma_s=cfg.sigma_s)


def config_order(cfg: Config | str) -> int:
    """N for the config: explicit for c0/c1, resolved from delta (Algorithm 1) for c2-c4."""
    from .order import epsilon_from_delta, estimate_order
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    if cfg.order is not None:
        return cfg.order
    k = config_kernel(cfg)
    return estimate_order(cfg.sigma_r, epsilon_from_delta(cfg.delta, k.w0, 128.0), 128.0).N0
