"""ORACLE — test infrastructure only (see nvol_oracle.py).

Render / macro-cell restatement of the reference (camera.py, transfer.py,
macrocell.py, render.py) on top of the C ray marcher in render.c.  Only tests
and bench.py's CPU legs may import this.
"""
from __future__ import annotations

import ctypes
import math

import numpy as np

import nvol_oracle as orc

TERMINATION = 1e-3  # render.py:28


def _lib():
    L = orc.lib()
    if not hasattr(L, "_render_sig"):
        P, I64, I32, F32, F64 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_float, ctypes.c_double
        L.orc_render_rm.argtypes = ([P, P, P, P, P, I64, I32, I32, I32] + [F32] * 5 + [P, I64, I64, I64, F64]
                                    + [F32] * 6 + [F64] * 3 + [I32, P, I64, I64, I64, P, P, P, P, P, I32, I32, P, P,
                                                               I32, I32, P, P, I32, P, P, I32, F32, I64, P])
        L.orc_render_rm.restype = I64
        L._render_sig = True
    return L


# ---------------------------------------------------------------- camera (camera.py)

def default_camera(dims, width=768, height=768):
    """camera.py:106-114 -> (eye, center, up, vfov, w, h)."""
    dx, dy, dz = (float(d) for d in dims)
    center = (dx / 2.0, dy / 2.0, dz / 2.0)
    reach = 1.6 * max(dx, dy, dz)
    look = np.array([1.0, 0.8, 1.1])
    look /= np.linalg.norm(look)
    eye = tuple(c + reach * l for c, l in zip(center, look))
    return dict(eye=eye, center=center, up=(0.0, 1.0, 0.0), vfov_deg=45.0, width=width, height=height)


def basis(cam):
    """camera.py:44-56."""
    e = np.asarray(cam["eye"], dtype=np.float64)
    c = np.asarray(cam["center"], dtype=np.float64)
    fwd = c - e
    fwd = fwd / np.linalg.norm(fwd)
    side = np.cross(fwd, np.asarray(cam["up"], dtype=np.float64))
    side = side / np.linalg.norm(side)
    return fwd, side, np.cross(side, fwd)


def camera_rays(cam):
    """camera.py:117-143."""
    w, h = cam["width"], cam["height"]
    idx = np.arange(w * h, dtype=np.float64)
    ii = idx % w
    jj = np.floor(idx / w)
    fwd, right, up = basis(cam)
    tan_half = math.tan(math.radians(cam["vfov_deg"]) * 0.5)
    aspect = w / h
    nx = ((ii + 0.5) / w * 2.0 - 1.0) * (tan_half * aspect)
    ny = (1.0 - (jj + 0.5) / h * 2.0) * tan_half
    d = fwd[None, :] + nx[:, None] * right[None, :] + ny[:, None] * up[None, :]
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    dirs = d.astype(np.float32)
    origins = np.broadcast_to(np.asarray(cam["eye"], dtype=np.float32), (dirs.shape[0], 3)).copy()
    return origins, dirs


def isect_batch(origins, dirs, hi):
    """render.py:225-243."""
    o = origins.astype(np.float64)
    d = dirs.astype(np.float64)
    h = np.asarray(hi, dtype=np.float64)
    with np.errstate(divide="ignore", invalid="ignore"):
        ta = (0.0 - o) / d
        tb = (h - o) / d
    lo = np.minimum(ta, tb)
    up = np.maximum(ta, tb)
    par = d == 0.0
    inside = (o >= 0.0) & (o <= h)
    lo[par & inside] = -np.inf
    up[par & inside] = np.inf
    lo[par & ~inside] = np.inf
    up[par & ~inside] = -np.inf
    t0 = np.maximum(lo.max(axis=1), 0.0)
    t1 = up.min(axis=1)
    return t0, t1, t1 > t0


# ---------------------------------------------------------------- transfer function (transfer.py)

def default_tf():
    """transfer.py:121-128."""
    return dict(colors=np.array([[0.0, 0.1, 0.2, 0.9], [0.5, 0.9, 0.4, 0.1], [1.0, 1.0, 0.9, 0.2]]),
                opacities=np.array([[0.0, 0.0], [0.3, 0.0], [0.6, 0.9], [1.0, 1.0]]), density_scale=2.0)


def tf_tables(tf):
    c = tf["colors"].astype(np.float32)
    o = tf["opacities"].astype(np.float32)
    return c[:, 0].copy(), np.ascontiguousarray(c[:, 1:]), o[:, 0].copy(), o[:, 1].copy()


# ---------------------------------------------------------------- macro-cells (macrocell.py)

def grid_dims(dims, ng):
    return tuple(-(-d // ng) for d in dims)


def ranges_from_array(norm, dims, ng):
    """macrocell.py:63-76 (bordered min/max)."""
    gx, gy, gz = grid_dims(dims, ng)
    dx, dy, dz = dims
    lo = np.full((gz, gy, gx), np.inf, dtype=np.float32)
    hi = np.full((gz, gy, gx), -np.inf, dtype=np.float32)
    for cz in range(gz):
        z0, z1 = max(cz * ng - 1, 0), min((cz + 1) * ng + 1, dz)
        for cy in range(gy):
            y0, y1 = max(cy * ng - 1, 0), min((cy + 1) * ng + 1, dy)
            for cx in range(gx):
                x0, x1 = max(cx * ng - 1, 0), min((cx + 1) * ng + 1, dx)
                block = norm[z0:z1, y0:y1, x0:x1]
                lo[cz, cy, cx] = block.min()
                hi[cz, cy, cx] = block.max()
    return lo, hi


def update_online(lo, hi, coords, targets, dims, ng):
    """macrocell.py:101-133 macrocell_update_online (in place on lo / hi)."""
    gx, gy, gz = grid_dims(dims, ng)
    d = np.array(dims, dtype=np.float32)
    s = coords.astype(np.float32) * d - np.float32(0.5)
    i0 = np.floor(s).astype(np.int64)
    vmax = np.array(dims, dtype=np.int64) - 1
    v_lo = np.clip(i0, 0, vmax)
    v_hi = np.clip(i0 + (s > i0.astype(np.float32)), 0, vmax)
    bound = np.array((gx, gy, gz), dtype=np.int64) - 1
    c_lo = np.clip((v_hi + ng - 1) // ng - 1, 0, bound)
    c_hi = np.clip((v_lo + 1) // ng, 0, bound)
    flat = np.concatenate([(iz * gy + iy) * gx + ix for iz in (c_lo[:, 2], c_hi[:, 2])
                           for iy in (c_lo[:, 1], c_hi[:, 1]) for ix in (c_lo[:, 0], c_hi[:, 0])])
    t = np.tile(targets.astype(np.float32), 8)
    np.minimum.at(lo.reshape(-1), flat, t)
    np.maximum.at(hi.reshape(-1), flat, t)


def voxel_centre_coords(dims):
    """macrocell.py:87-94: centres computed in float64, then cast to float32."""
    dx, dy, dz = dims
    zz, yy, xx = np.meshgrid(np.arange(dz), np.arange(dy), np.arange(dx), indexing="ij")
    return np.stack([(xx.ravel() + 0.5) / dx, (yy.ravel() + 0.5) / dy, (zz.ravel() + 0.5) / dz],
                    axis=1).astype(np.float32)


def macrocell_from_model(model: "orc.OracleModel", dims, ng):
    """macrocell.py:84-98."""
    vals = model.eval_fused(voxel_centre_coords(dims))
    dx, dy, dz = dims
    return ranges_from_array(np.clip(vals, 0.0, 1.0).reshape(dz, dy, dx), dims, ng)


def set_tf(lo_arr, hi_arr, tf):
    """macrocell.py:136-156 -> mu_max (f32)."""
    lo = np.clip(lo_arr.reshape(-1).astype(np.float64), 0.0, 1.0)
    hi = np.clip(hi_arr.reshape(-1).astype(np.float64), 0.0, 1.0)
    touched = lo_arr.reshape(-1) <= hi_arr.reshape(-1)
    pv, pa = tf["opacities"][:, 0], tf["opacities"][:, 1]
    best = np.maximum(np.interp(lo, pv, pa), np.interp(hi, pv, pa))
    interior = (pv[None, :] > lo[:, None]) & (pv[None, :] < hi[:, None])
    if interior.any():
        best = np.maximum(best, np.where(interior, pa[None, :], -np.inf).max(axis=1))
    mu = np.where(touched, best * tf["density_scale"], 0.0)
    return mu.reshape(lo_arr.shape).astype(np.float32)


# ---------------------------------------------------------------- render (render.py)

def render(field, tf, cam, mode="raymarch", use_macrocells=True, mu=None, ng=64, step_size=1.0, max_step=64.0,
           step_exponent=2.0, k_batch=8, light_direction=(-0.57735026919, -0.57735026919, -0.57735026919),
           background=(1.0, 1.0, 1.0), ambient=0.2, skip_empty=True, dims=None):
    """render_reference (render.py:347-380) with the oracle field.  `field` is an
    OracleModel or a (dz,dy,dx) float32 normalised grid.  Returns (img (H,W,3), evals)."""
    L = _lib()
    is_grid = isinstance(field, np.ndarray)
    if dims is None:
        dims = (field.shape[2], field.shape[1], field.shape[0]) if is_grid else None
    hx, hy, hz = (float(d) for d in dims)
    origins, dirs = camera_rays(cam)
    t0, t1, hit = isect_batch(origins, dirs, (hx, hy, hz))
    o, d = np.ascontiguousarray(origins[hit]), np.ascontiguousarray(dirs[hit])
    t0h, t1h = np.ascontiguousarray(t0[hit]), np.ascontiguousarray(t1[hit])
    pixels = np.nonzero(hit)[0].astype(np.int64)
    w, h = cam["width"], cam["height"]
    img = np.empty((w * h, 3), dtype=np.float32)
    bg = tuple(np.float32(c) for c in background)
    img[:] = bg
    ln = np.asarray(light_direction, dtype=np.float64)
    ln = ln / np.linalg.norm(ln)
    sd = tuple(np.float32(-c) for c in ln)
    if use_macrocells:
        mu_arr = np.ascontiguousarray(mu, dtype=np.float32)
        gz, gy, gx = mu_arr.shape
        ngf = float(ng)
    else:
        mu_arr = np.zeros((1, 1, 1), dtype=np.float32)
        gz = gy = gx = 1
        ngf = 1.0
    cv, crgb, ov, oa = tf_tables(tf)
    ds = np.float32(tf["density_scale"])
    P = orc._p
    if is_grid:
        norm = np.ascontiguousarray(field, dtype=np.float32)
        dummy64 = np.zeros(1, np.int64)
        args_field = (1, P(norm), norm.shape[2], norm.shape[1], norm.shape[0], P(np.zeros(1, np.float32)),
                      P(dummy64), P(np.ones(1, np.int64)), P(np.ones(1, np.int64)), P(np.ones(1, np.uint8)), 1, 1,
                      P(np.zeros(1, np.float32)), P(np.array([1, 1], np.int32)), 1, 0)
        keep = (norm, dummy64)
    else:
        res, ent, dense, off = orc.level_tables(field.spec)
        flat = np.concatenate([wm.ravel() for wm in field.weights]).astype(np.float32)
        widths = np.array([field.weights[0].shape[1]] + [wm.shape[0] for wm in field.weights], dtype=np.int32)
        args_field = (0, P(np.zeros(1, np.float32)), 1, 1, 1, P(field.params), P(off), P(res), P(ent), P(dense),
                      field.spec.n_levels, field.spec.n_features_per_level, P(flat), P(widths), len(field.weights),
                      int(field.relu_out))
        keep = (res, ent, dense, off, flat, widths)
    evals = L.orc_render_rm(P(o), P(d), P(t0h), P(t1h), P(pixels), o.shape[0], int(mode == "raymarch_shadow"),
                            int(use_macrocells), int(skip_empty), np.float32(step_size), np.float32(max_step),
                            np.float32(step_exponent), np.float32(TERMINATION), np.float32(ambient), P(mu_arr), gx, gy,
                            gz, ngf, sd[0], sd[1], sd[2], bg[0], bg[1], bg[2], hx, hy, hz, *args_field, P(cv), P(crgb),
                            len(cv), P(ov), P(oa), len(ov), ds, int(k_batch), P(img))
    del keep
    return img.reshape(h, w, 3), int(evals)
