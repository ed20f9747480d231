"""Multi-resolution grid encoder (hash grid / dense grid) on the B200.

Mirror of the reference's encoding.py (/root/reference/pkg/src/neuralvol/
encoding.py): same config validation, table layout (level-major,
entry-major, feature-minor), initialisation stream and method names.  Tables
live in device memory as torch tensors; encode / encode_backward run the
sm_100a kernels of csrc/encoder.cu through the C ABI.  Float32 encodings,
slot indices and corner weights are bit-identical to the reference.

The fixed-function encoders (identity / frequency / one-blob,
encoding.py:112-142) are accepted by EncoderConfig for config parity but are
outside the B200 hot path: make_encoder raises ConfigError for them.
"""
from __future__ import annotations

from contextlib import contextmanager

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._tensor import out, to_device, torch_dtype
from .errors import ConfigError

HASH_PRIMES = (1, 2654435761, 805459861)           # encoding.py:22
GRID_KINDS = ("densegrid", "hashgrid")
KINDS = ("identity", "frequency", "oneblob") + GRID_KINDS
FEATURE_INIT_SCALE = 1e-4                          # encoding.py:27

_deterministic = False


def set_deterministic(flag: bool) -> None:
    """Bitwise run-to-run repeatability (the reference's SPEC.md:197,286,785):
    encoder backward scatters go through the order-preserving kernel
    (bit-identical to the reference's serial scatter) instead of float atomics,
    and training runs on the fp32 SIMT engine with every reduction ordered
    (nvol_set_deterministic: split-K dW GEMMs, loss sum)."""
    global _deterministic
    _deterministic = bool(flag)
    _lib.load().nvol_set_deterministic(int(_deterministic))


def deterministic() -> bool:
    return _deterministic


@contextmanager
def deterministic_mode(flag: bool = True):
    """set_deterministic(flag) for the duration of a block, then the previous mode."""
    prev = _deterministic
    set_deterministic(flag)
    try:
        yield
    finally:
        set_deterministic(prev)


@dataclass(frozen=True)
class EncoderConfig:
    """encoding.py:30-68."""
    kind: str = "hashgrid"
    n_levels: int = 8
    n_features_per_level: int = 4
    log2_hashmap_size: int = 15
    base_resolution: int = 4
    per_level_scale: float = 2.0
    n_frequencies: int = 32
    n_bins: int = 64

    def __post_init__(self) -> None:
        if self.kind not in KINDS:
            raise ConfigError(f"unknown encoder kind {self.kind!r}; expected one of {KINDS}")
        if self.kind in GRID_KINDS:
            if self.n_levels < 1:
                raise ConfigError("grid encoders require n_levels >= 1")
            if self.n_features_per_level not in (1, 2, 4, 8):
                raise ConfigError(f"n_features_per_level must be in {{1,2,4,8}}, got {self.n_features_per_level}")
            if not 10 <= self.log2_hashmap_size <= 24:
                raise ConfigError(f"log2_hashmap_size must lie in [10,24], got {self.log2_hashmap_size}")
            if self.base_resolution < 1:
                raise ConfigError("base_resolution must be >= 1")
            if self.per_level_scale <= 0:
                raise ConfigError("per_level_scale must be > 0")
        if self.kind == "frequency" and self.n_frequencies < 1:
            raise ConfigError("frequency encoder requires n_frequencies >= 1")
        if self.kind == "oneblob" and self.n_bins < 1:
            raise ConfigError("oneblob encoder requires n_bins >= 1")

    @property
    def out_width(self) -> int:
        if self.kind == "identity":
            return 3
        if self.kind == "frequency":
            return 6 * self.n_frequencies
        if self.kind == "oneblob":
            return 3 * self.n_bins
        return self.n_features_per_level * self.n_levels


def level_resolution(config: EncoderConfig, level: int) -> int:
    """R_l = floor(base_resolution * per_level_scale^level)  (encoding.py:71-75)."""
    if not 0 <= level < config.n_levels:
        raise ConfigError(f"level {level} out of range [0, {config.n_levels})")
    return int(math.floor(config.base_resolution * config.per_level_scale ** level))


def _check_coords_shape(p: torch.Tensor) -> torch.Tensor:
    if p.ndim == 1:
        p = p[None, :]
    if p.ndim != 2 or p.shape[1] != 3:
        raise ConfigError(f"coordinates must be (B,3), got shape {tuple(p.shape)}")
    return p


class Encoder:
    """Base class (encoding.py:87-109)."""

    def __init__(self, config: EncoderConfig, dtype=np.float32):
        self.config = config
        self.dtype = np.dtype(dtype)

    @property
    def out_width(self) -> int:
        return self.config.out_width


class GridEncoder(Encoder):
    """Dense or hashed multi-resolution feature grids with trilinear blending
    (encoding.py:145-226).  `params` / `param_grads` are device tensors."""

    def __init__(self, config: EncoderConfig, dtype=np.float32, rng: np.random.Generator | None = None,
                 device=None):
        super().__init__(config, dtype)
        if config.kind not in GRID_KINDS:
            raise ConfigError(f"GridEncoder needs a grid kind, got {config.kind!r}")
        if config.n_levels > 32:
            raise ConfigError("the B200 encoder supports at most 32 levels")
        n = config.n_features_per_level
        table_size = 1 << config.log2_hashmap_size
        self.level_resolutions = np.array([level_resolution(config, l) for l in range(config.n_levels)],
                                          dtype=np.int64)
        dense_sizes = (self.level_resolutions + 1) ** 3
        if config.kind == "densegrid":
            self.level_entries = dense_sizes.copy()
        else:
            self.level_entries = np.minimum(dense_sizes, table_size)
        self.level_offsets = np.concatenate([[0], np.cumsum(self.level_entries * n)])[:-1].astype(np.int64)
        total = int((self.level_entries * n).sum())
        rng = rng if rng is not None else np.random.default_rng(0)
        # same draws as encoding.py:167-168 (host RNG, then one upload)
        init = rng.uniform(-FEATURE_INIT_SCALE, FEATURE_INIT_SCALE, size=total).astype(self.dtype)
        dev = device if device is not None else _lib.device()
        self.params = torch.from_numpy(init).to(dev)
        self.param_grads = torch.zeros(total, dtype=torch_dtype(self.dtype), device=dev)
        self._dense = np.array([self._level_dense(l) for l in range(config.n_levels)], dtype=np.uint8)
        self._c_tables = (_lib.host_i64(self.level_offsets), _lib.host_i64(self.level_resolutions),
                          _lib.host_i64(self.level_entries), _lib.host_u8(self._dense))

    @property
    def n_params(self) -> int:
        return int(self.params.numel())

    def _level_dense(self, l: int) -> bool:
        return bool((self.level_resolutions[l] + 1) ** 3 <= self.level_entries[l])

    def kernel_tables(self):
        """Level tables in the layout the kernels expect (encoding.py:174-177)."""
        return self.level_resolutions, self.level_entries, self._dense.copy(), self.level_offsets

    def c_tables(self):
        """(level_off, level_res, level_entries, level_dense) as ctypes host arrays."""
        return self._c_tables

    def encode_device(self, p: torch.Tensor, want_cache: bool = False, check_nan: bool = True):
        """Device tensors in, device tensors out: (feats, idx_cache|None, w_cache|None)."""
        p = _check_coords_shape(p)
        if p.dtype != self.params.dtype:
            p = p.to(self.params.dtype)
        p = p.contiguous()
        if check_nan and p.numel() and bool(torch.isnan(p).any()):
            raise ConfigError("encode input contains NaN")
        b, m, n = p.shape[0], self.config.n_levels, self.config.n_features_per_level
        feats = torch.empty((b, m * n), dtype=self.params.dtype, device=p.device)
        idx = torch.empty((b, m, 8), dtype=torch.int64, device=p.device) if want_cache else None
        w = torch.empty((b, m, 8), dtype=self.params.dtype, device=p.device) if want_cache else None
        off, res, ent, dense = self._c_tables
        _lib.call("nvol_grid_encode_fwd", _lib.ptr(p), b, _lib.ptr(self.params), off, res, ent, dense, m, n,
                  _lib.ptr(idx), _lib.ptr(w), _lib.ptr(feats), self.params.element_size(), _lib.stream())
        return feats, idx, w

    def encode(self, p):
        """Feature matrix (B, m*n) for coordinates (B,3) (encoding.py:203-213)."""
        t, host = to_device(p, self.dtype)
        feats, _, _ = self.encode_device(t)
        return out(feats, host)

    def encode_backward(self, p, dl_dfeat) -> None:
        """Accumulate dL/dparams into param_grads (encoding.py:215-226)."""
        t, _ = to_device(p, self.dtype)
        t = _check_coords_shape(t)
        g, _ = to_device(dl_dfeat, self.dtype)
        if tuple(g.shape) != (t.shape[0], self.out_width):
            raise ConfigError(f"gradient shape {tuple(g.shape)} does not match ({t.shape[0]}, {self.out_width})")
        if t.numel() and bool(torch.isnan(t).any()):
            raise ConfigError("encode input contains NaN")
        self.backward_device(t.contiguous(), g.contiguous())

    def backward_device(self, p: torch.Tensor, dl_dfeat: torch.Tensor) -> None:
        off, res, ent, dense = self._c_tables
        det = 1 if (_deterministic and self.params.dtype == torch.float32) else 0
        _lib.call("nvol_grid_encode_bwd_coords", _lib.ptr(p), _lib.ptr(dl_dfeat), p.shape[0], off, res, ent,
                  dense, self.config.n_levels, self.config.n_features_per_level, _lib.ptr(self.param_grads),
                  self.params.element_size(), det, _lib.stream())

    def backward_from_cache(self, dl_dfeat: torch.Tensor, idx_cache: torch.Tensor, w_cache: torch.Tensor) -> None:
        """_kernels.py:82-92 grid_encode_bwd over the forward caches."""
        b, m, _ = idx_cache.shape
        _lib.call("nvol_grid_encode_bwd", _lib.ptr(dl_dfeat.contiguous()), _lib.ptr(idx_cache),
                  _lib.ptr(w_cache), b, m, self.config.n_features_per_level, _lib.ptr(self.param_grads),
                  self.params.element_size(), _lib.stream())


def hash_index(level_entries: int, resolution: int, vertex, dense: bool | None = None) -> int:
    """Slot of one lattice vertex (encoding.py:229-234); host-side inspection helper."""
    vx, vy, vz = (int(v) for v in vertex)
    if dense is None:
        dense = (resolution + 1) ** 3 <= level_entries
    if dense:
        r1 = resolution + 1
        return (vz * r1 + vy) * r1 + vx
    m32 = 0xFFFFFFFF
    h = ((vx * HASH_PRIMES[0]) & m32) ^ ((vy * HASH_PRIMES[1]) & m32) ^ ((vz * HASH_PRIMES[2]) & m32)
    return (h & m32) % level_entries


def corner_weights(fr: np.ndarray) -> np.ndarray:
    """The 8 trilinear weights for fractional offsets fr (B,3) (encoding.py:249-260);
    host-side inspection helper."""
    fr = np.atleast_2d(fr)
    w = np.empty((fr.shape[0], 8), dtype=fr.dtype)
    for c in range(8):
        ox, oy, oz = (c >> 0) & 1, (c >> 1) & 1, (c >> 2) & 1
        w[:, c] = ((fr[:, 0] if ox else 1 - fr[:, 0]) * (fr[:, 1] if oy else 1 - fr[:, 1])
                   * (fr[:, 2] if oz else 1 - fr[:, 2]))
    return w


def make_encoder(config: EncoderConfig, dtype=np.float32, rng: np.random.Generator | None = None) -> GridEncoder:
    """encoding.py:263-270 restricted to the grid kinds (the B200 hot path)."""
    if config.kind not in GRID_KINDS:
        raise ConfigError(f"encoder kind {config.kind!r} is outside the B200 hot path "
                          "(hashgrid / densegrid only)")
    return GridEncoder(config, dtype, rng)


def encode(encoder: GridEncoder, p):
    """Feature vector(s) for p; accepts one coordinate (3,) or a batch (B,3) (encoding.py:273-278)."""
    single = np.ndim(p) == 1 if not isinstance(p, torch.Tensor) else p.ndim == 1
    o = encoder.encode(p[None, :] if single else p)
    return o[0] if single else o


def encode_backward(encoder: GridEncoder, p, dl_dfeat) -> None:
    """encoding.py:281-287."""
    if (p.ndim if isinstance(p, torch.Tensor) else np.ndim(p)) == 1:
        p = p[None, :]
        dl_dfeat = dl_dfeat[None, :]
    encoder.encode_backward(p, dl_dfeat)
