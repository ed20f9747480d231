"""The reference's numba FFI (/root/reference/pkg/src/neuralvol/_kernels.py) served by
libnvol.so: same functions, same caller-allocated numpy outputs, each call one
H2D of the inputs, the C-ABI launch, one D2H of the outputs (include/nvol.h).

    grid_encode_fwd   -> nvol_grid_encode_fwd   (_kernels.py:31-79)
    grid_encode_bwd   -> nvol_grid_encode_bwd   (_kernels.py:82-92)
    field_eval_model  -> nvol_field_eval_exact  (_kernels.py:154-176)
"""
from __future__ import annotations

import numpy as np
import torch

from paper_2207_11620_b200 import _lib


def _dev(a, dtype=None):
    t = torch.from_numpy(np.ascontiguousarray(a, dtype=dtype))
    return t.to(_lib.device())


def _tables(level_off, level_res, level_entries, level_dense):
    return (_lib.host_i64(level_off), _lib.host_i64(level_res), _lib.host_i64(level_entries),
            _lib.host_u8(level_dense))


def grid_encode_fwd(coords, params, level_off, level_res, level_entries, level_dense, n_feat, idx_cache, w_cache,
                    out):
    eb = _lib.dtype_bytes(out.dtype)
    dt = out.dtype
    c, p = _dev(coords, dt), _dev(params, dt)
    idx = torch.empty(idx_cache.shape, dtype=torch.int64, device=c.device)
    w = torch.empty(w_cache.shape, dtype=c.dtype, device=c.device)
    o = torch.empty(out.shape, dtype=c.dtype, device=c.device)
    _lib.call("nvol_grid_encode_fwd", _lib.ptr(c), c.shape[0], _lib.ptr(p),
              *_tables(level_off, level_res, level_entries, level_dense), len(level_res), int(n_feat),
              _lib.ptr(idx), _lib.ptr(w), _lib.ptr(o), eb, _lib.stream())
    idx_cache[...] = idx.cpu().numpy()
    w_cache[...] = w.cpu().numpy()
    out[...] = o.cpu().numpy()


def grid_encode_bwd(dl_dfeat, idx_cache, w_cache, n_feat, grad_out):
    eb = _lib.dtype_bytes(grad_out.dtype)
    dt = grad_out.dtype
    d, idx, w, g = _dev(dl_dfeat, dt), _dev(idx_cache, np.int64), _dev(w_cache, dt), _dev(grad_out, dt)
    b, m = idx_cache.shape[0], idx_cache.shape[1]
    _lib.call("nvol_grid_encode_bwd", _lib.ptr(d), _lib.ptr(idx), _lib.ptr(w), b, m, int(n_feat), _lib.ptr(g), eb,
              _lib.stream())
    grad_out[...] = g.cpu().numpy()


def field_eval_model(coords, params, level_off, level_res, level_entries, level_dense, n_feat, weights, relu_out,
                     out):
    c, p = _dev(coords, np.float32), _dev(params, np.float32)
    widths = [int(weights[0].shape[1])] + [int(w.shape[0]) for w in weights]
    wf = _dev(np.concatenate([np.asarray(w, np.float32).ravel() for w in weights]))
    o = torch.empty(c.shape[0], dtype=torch.float32, device=c.device)
    _lib.call("nvol_field_eval_exact", _lib.ptr(c), c.shape[0], _lib.ptr(p),
              *_tables(level_off, level_res, level_entries, level_dense), len(level_res), int(n_feat),
              _lib.ptr(wf), _lib.host_i32(widths), len(weights), int(bool(relu_out)), _lib.ptr(o), _lib.stream())
    out[...] = o.cpu().numpy()
