"""Scalar tracking helpers of the reference (tracking.py) for tests and inspection.

adaptive_step and correct_opacity evaluate the ray marcher's own device formulas (one
nvol_march_formula launch), so what is inspected here is what renders.  woodcock and
woodcock_dda are host delta-tracking estimators over a Python callable sigma(t) -- the
statistical oracles the reference's tests drive the device path tracer against (the path
tracer itself runs delta tracking on the device, render.cu pt_*).
"""
from __future__ import annotations

import math

import numpy as np
import torch

from . import _lib
from .errors import ConfigError


def _formula(which: int, x: float, a: float, b: float, c: float = 0.0) -> np.float32:
    dev = _lib.device()
    t = torch.tensor([x], dtype=torch.float32, device=dev)
    o = torch.empty(1, dtype=torch.float32, device=dev)
    _lib.call("nvol_march_formula", which, _lib.ptr(t), 1, float(a), float(b), float(c), _lib.ptr(o), _lib.stream())
    return np.float32(o.item())


def adaptive_step(mu_max: float, s1: float, s2: float, p: float) -> np.float32:
    """Step length between s1 (dense regions) and s2 (empty regions) (tracking.py:21-26)."""
    return _formula(0, mu_max, s1, s2, p)


def correct_opacity(alpha: float, sbar: float, s1: float) -> np.float32:
    """Opacity resampled from step s1 to step sbar: 1 - (1 - alpha)^(sbar / s1) (tracking.py:29-31)."""
    return _formula(1, alpha, sbar, s1)


def woodcock(sigma, mu_max: float, t_min: float, t_max: float, rng):
    """First real collision of the extinction sigma(t) on [t_min, t_max] by delta tracking against
    the majorant mu_max (tracking.py:46-66), or None if the ray leaves the interval."""
    if not mu_max > 0.0:
        return None
    t = float(t_min)
    while True:
        t -= math.log(1.0 - float(rng.random())) / mu_max
        if t >= t_max:
            return None
        s = float(sigma(t))
        if s > mu_max * (1.0 + 1e-6):
            raise ConfigError(f"majorant violated: sigma({t}) = {s} > {mu_max}")
        if float(rng.random()) * mu_max < s:
            return t


def woodcock_dda(grid, sigma, ray, rng):
    """woodcock, walking the macro-cells (device DDA, macrocell.dda_traverse) so each cell's
    segment is tracked against its own majorant grid.mu_max[cz, cy, cx] (tracking.py:69-107)."""
    from .macrocell import dda_traverse
    origin, direction = ray
    mu = grid.mu_max.cpu().numpy() if isinstance(grid.mu_max, torch.Tensor) else np.asarray(grid.mu_max)
    hit = []

    def visit(cell, s0, s1):
        t = woodcock(sigma, float(mu[cell[2], cell[1], cell[0]]), s0, s1, rng)
        if t is not None:
            hit.append(t)
            return False
        return True

    dda_traverse(grid, origin, direction, visit)
    return hit[0] if hit else None
