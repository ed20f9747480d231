"""Macro-cell acceleration grid (macrocell.py of the reference) on the device.

Per-cell value ranges (bordered min/max, macrocell.py:63-76) and exact
opacity majorants (macrocell.py:136-156) are computed by csrc/render.cu
kernels; `macrocell_from_model` decodes Phi at every voxel centre with the
exact evaluator (float64 centre coordinates, as macrocell.py:87-94) and
reduces on the device.  Arrays (`value_lo`, `value_hi`, `mu_max`) are device
tensors shaped (gz, gy, gx).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .errors import ConfigError
from .transfer import TransferFunction

DEFAULT_CELL_SIZE = 64


@dataclass
class MacroCellGrid:
    """macrocell.py:27-55."""
    vol_dims: tuple
    n_g: int = DEFAULT_CELL_SIZE
    value_lo: object = field(default=None, repr=False)
    value_hi: object = field(default=None, repr=False)
    mu_max: object = field(default=None, repr=False)

    def __post_init__(self) -> None:
        if self.n_g < 1:
            raise ConfigError(f"macro-cell size must be >= 1, got {self.n_g}")
        dx, dy, dz = (int(d) for d in self.vol_dims)
        if min(dx, dy, dz) < 1:
            raise ConfigError(f"bad volume dims {self.vol_dims}")
        self.vol_dims = (dx, dy, dz)
        gx, gy, gz = self.grid_dims
        shape = (gz, gy, gx)
        dev = _lib.device()
        if self.value_lo is None:
            self.value_lo = torch.full(shape, float("inf"), dtype=torch.float32, device=dev)
            self.value_hi = torch.full(shape, float("-inf"), dtype=torch.float32, device=dev)
        if self.mu_max is None:
            self.mu_max = torch.zeros(shape, dtype=torch.float32, device=dev)
        for name in ("value_lo", "value_hi", "mu_max"):
            arr = getattr(self, name)
            if not isinstance(arr, torch.Tensor):
                setattr(self, name, torch.as_tensor(np.asarray(arr, dtype=np.float32), device=dev))
            if tuple(getattr(self, name).shape) != shape:
                raise ConfigError(f"cell array shape {tuple(getattr(self, name).shape)} != grid {shape}")

    @property
    def grid_dims(self):
        return tuple(-(-d // self.n_g) for d in self.vol_dims)


def macrocell_empty(dims, n_g: int = DEFAULT_CELL_SIZE) -> MacroCellGrid:
    return MacroCellGrid(vol_dims=tuple(dims), n_g=n_g)


def _ranges(vals: torch.Tensor, dims, n_g: int, clip: bool) -> MacroCellGrid:
    grid = macrocell_empty(dims, n_g)
    dx, dy, dz = grid.vol_dims
    _lib.call("nvol_macrocell_ranges", _lib.ptr(vals.contiguous()), dx, dy, dz, n_g, int(clip),
              _lib.ptr(grid.value_lo), _lib.ptr(grid.value_hi), _lib.stream())
    return grid


def macrocell_build(fld, n_g: int = DEFAULT_CELL_SIZE) -> MacroCellGrid:
    """Per-cell min/max (with border) of a dense volume (macrocell.py:79-81)."""
    return _ranges(fld.normalized, fld.meta.dims, n_g, clip=False)


def macrocell_from_model(model, n_g: int = DEFAULT_CELL_SIZE, chunk: int = 0) -> MacroCellGrid:
    """Ranges from the model decoded at voxel centres (macrocell.py:84-98).

    A NeuralModel is decoded on the device; any other object with the reference's
    `dims` + `eval_fused(coords)` protocol is evaluated through that method, in chunks of
    `chunk` voxel centres computed exactly as the reference does, and the ranges are
    taken on the device."""
    from .model import NeuralModel
    from .trainer import decode_brick
    dx, dy, dz = model.dims
    if not isinstance(model, NeuralModel):
        step = int(chunk) if chunk else 262144
        zz, yy, xx = np.meshgrid(np.arange(dz), np.arange(dy), np.arange(dx), indexing="ij")
        coords = np.stack([(xx.ravel() + 0.5) / dx, (yy.ravel() + 0.5) / dy, (zz.ravel() + 0.5) / dz],
                          axis=1).astype(np.float32)
        vals = np.empty(dx * dy * dz, dtype=np.float32)
        for s in range(0, coords.shape[0], step):
            v = model.eval_fused(coords[s:s + step])
            vals[s:s + step] = v.cpu().numpy() if isinstance(v, torch.Tensor) else np.asarray(v, np.float32)
        return _ranges(torch.from_numpy(vals.reshape(dz, dy, dx)).to(_lib.device()), (dx, dy, dz), n_g, clip=True)
    vals = torch.empty((dz, dy, dx), dtype=torch.float32, device=model.flat_params.device)
    decode_brick(model, (dx, dy, dz), 0, dz, vals, mode="centres64")
    return _ranges(vals, (dx, dy, dz), n_g, clip=True)


def macrocell_update_online(grid: MacroCellGrid, batch) -> None:
    """Widen cell ranges with a training batch (macrocell.py:101-133), on the device
    (nvol_macrocell_update_online: int-ordered atomic min / max, bit-exact)."""
    c = batch.coords if isinstance(batch.coords, torch.Tensor) else torch.as_tensor(np.asarray(batch.coords))
    t = batch.targets if isinstance(batch.targets, torch.Tensor) else torch.as_tensor(np.asarray(batch.targets))
    n = int(c.shape[0])
    if n == 0:
        return
    dev = grid.value_lo.device
    c = c.to(dev, torch.float32).contiguous()
    t = t.to(dev, torch.float32).contiguous()
    dx, dy, dz = grid.vol_dims
    gx, gy, gz = grid.grid_dims
    _lib.call("nvol_macrocell_update_online", _lib.ptr(c), _lib.ptr(t), n, dx, dy, dz, _lib.ptr(grid.value_lo),
              _lib.ptr(grid.value_hi), gx, gy, gz, grid.n_g, _lib.stream())


class OnlineMacrocells:
    """Training tap `tap(batch) = macrocell_update_online(grid, batch)` (the
    reference's live session, service.py:279).  trainer.train recognises it and
    fuses the update into the device sampler kernel (no extra launch)."""

    def __init__(self, grid: MacroCellGrid):
        self.grid = grid

    def __call__(self, batch) -> None:
        macrocell_update_online(self.grid, batch)


def macrocell_set_tf(grid: MacroCellGrid, tf: TransferFunction) -> None:
    """Exact per-cell majorant for the current TF (macrocell.py:136-156)."""
    pv = np.ascontiguousarray(tf.opacity_points[:, 0], dtype=np.float64)
    pa = np.ascontiguousarray(tf.opacity_points[:, 1], dtype=np.float64)
    cv = (np.ctypeslib.as_ctypes(pv), np.ctypeslib.as_ctypes(pa))
    _lib.call("nvol_macrocell_set_tf", _lib.ptr(grid.value_lo), _lib.ptr(grid.value_hi), grid.value_lo.numel(),
              cv[0], cv[1], len(pv), float(tf.density_scale), _lib.ptr(grid.mu_max), _lib.stream())


def dda_traverse(grid: MacroCellGrid, origin, direction, visitor) -> None:
    """Walk the cells pierced by the ray inside the volume box, front to back (macrocell.py:159-181).

    visitor(cell_xyz (3,) int64, s_enter, s_exit) -> bool; returning False stops the walk.  The
    segments tile [t_min, t_max] of the ray / volume intersection exactly.  The walk runs on the
    device (nvol_dda_collect), in float64 like the marcher's cell stepping."""
    from .camera import intersect_aabb
    dx, dy, dz = grid.vol_dims
    hit = intersect_aabb(origin, direction, (dx, dy, dz))
    if hit is None:
        return
    t0, t1 = hit
    gx, gy, gz = grid.grid_dims
    cap = gx + gy + gz + 4
    dev = _lib.device()
    cells = torch.empty((cap, 3), dtype=torch.int64, device=dev)
    ts = torch.empty((cap, 2), dtype=torch.float64, device=dev)
    count = torch.zeros(1, dtype=torch.int64, device=dev)
    ray = (ctypes.c_double * 6)(*[float(x) for x in (*origin, *direction)])
    _lib.call("nvol_dda_collect", ray, float(t0), float(t1), float(grid.n_g), gx, gy, gz, cap, _lib.ptr(cells),
              _lib.ptr(ts), _lib.ptr(count), _lib.stream())
    n = int(count.item())
    c, t = cells[:n].cpu().numpy(), ts[:n].cpu().numpy()
    for i in range(n):
        if visitor(c[i], float(t[i, 0]), float(t[i, 1])) is False:
            return
