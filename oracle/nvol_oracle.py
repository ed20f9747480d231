"""ORACLE — test infrastructure only.

CPU restatement of the reference's hash-grid hot path
(/root/reference/pkg/src/neuralvol, arXiv 2207.11620 CPU reference).  Only
tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
leg may import this module; the product package never does.

Split of work:
  * the reference's numba kernels (encoder fwd/bwd, fused field evaluator,
    trilinear GT lookup) and its dense Adam are restated in C (kernels.c,
    compiled with -ffp-contract=off, bit-identical to the reference);
  * the reference's BLAS-backed MLP and float64 loss are restated here with
    the same numpy operations (network.py:61-114), i.e. the same OpenBLAS
    sgemm calls the reference makes;
  * numpy's PCG64 (the reference's third-party coordinate generator,
    sampler.py:54-55, numpy 2.3.5) is restated in C and checked against
    numpy itself.

Pinned against golden vectors produced by importing the reference in the build
container (oracle/gen_golden.py -> tests/golden/*.npz).
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_LIB_PATH = _HERE / "build" / "liboracle.so"
_lib = None

HASH_PRIMES = (1, 2654435761, 805459861)  # encoding.py:22
FEATURE_INIT_SCALE = 1e-4                  # encoding.py:27


def build() -> Path:
    subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not _LIB_PATH.exists():
            build()
        L = ctypes.CDLL(str(_LIB_PATH))
        P = ctypes.c_void_p
        i64, i32, f32, u64 = ctypes.c_int64, ctypes.c_int, ctypes.c_float, ctypes.c_uint64
        L.orc_grid_encode_fwd.argtypes = [P, i64, P, P, P, P, P, i32, i32, P, P, P]
        L.orc_grid_encode_bwd.argtypes = [P, P, P, i64, i32, i32, P]
        L.orc_field_eval_model.argtypes = [P, i64, P, P, P, P, P, i32, i32, P, P, i32, i32, P]
        L.orc_adam_f32.argtypes = [P, P, P, P, i64] + [f32] * 9
        L.orc_pcg64_random_f32.argtypes = [u64, u64, u64, u64, u64, i64, P]
        L.orc_trilinear.argtypes = [P, i64, i64, i64, P, i64, i32, P]
        L.orc_num_threads.restype = i32
        L.orc_set_threads.argtypes = [i32]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def num_threads() -> int:
    return int(lib().orc_num_threads())


def set_threads(n: int) -> None:
    lib().orc_set_threads(int(n))


# ---------------------------------------------------------------- encoder tables

@dataclass(frozen=True)
class GridSpec:
    """encoding.py:30-68 EncoderConfig restricted to the grid kinds."""
    kind: str = "hashgrid"
    n_levels: int = 8
    n_features_per_level: int = 4
    log2_hashmap_size: int = 15
    base_resolution: int = 4
    per_level_scale: float = 2.0

    @property
    def out_width(self) -> int:
        return self.n_levels * self.n_features_per_level


def level_tables(spec: GridSpec):
    """encoding.py:71-75 level_resolution, encoding.py:157-177 entries/offsets/dense."""
    n = spec.n_features_per_level
    res = np.array([int(math.floor(spec.base_resolution * spec.per_level_scale ** l))
                    for l in range(spec.n_levels)], dtype=np.int64)
    dense_sizes = (res + 1) ** 3
    if spec.kind == "densegrid":
        entries = dense_sizes.copy()
    else:
        entries = np.minimum(dense_sizes, 1 << spec.log2_hashmap_size)
    offsets = np.concatenate([[0], np.cumsum(entries * n)])[:-1].astype(np.int64)
    dense = ((res + 1) ** 3 <= entries).astype(np.uint8)
    return res, entries, dense, offsets


def grid_encode_fwd(coords, params, spec: GridSpec, want_cache: bool = True):
    """_kernels.py:31-79 grid_encode_fwd -> (out, idx_cache, w_cache)."""
    coords = np.ascontiguousarray(coords, dtype=np.float32)
    params = np.ascontiguousarray(params, dtype=np.float32)
    res, entries, dense, off = level_tables(spec)
    b, m, n = coords.shape[0], spec.n_levels, spec.n_features_per_level
    out = np.empty((b, m * n), dtype=np.float32)
    idx = np.empty((b, m, 8), dtype=np.int64) if want_cache else None
    w = np.empty((b, m, 8), dtype=np.float32) if want_cache else None
    lib().orc_grid_encode_fwd(_p(coords), b, _p(params), _p(off), _p(res), _p(entries), _p(dense),
                              m, n, _p(idx) if want_cache else None,
                              _p(w) if want_cache else None, _p(out))
    return out, idx, w


def grid_encode_bwd(dl_dfeat, idx_cache, w_cache, n_feat: int, grad_out: np.ndarray) -> None:
    """_kernels.py:82-92 grid_encode_bwd (accumulates into grad_out)."""
    dl = np.ascontiguousarray(dl_dfeat, dtype=np.float32)
    b, m, _ = idx_cache.shape
    assert grad_out.dtype == np.float32 and grad_out.flags.c_contiguous
    lib().orc_grid_encode_bwd(_p(dl), _p(np.ascontiguousarray(idx_cache)),
                              _p(np.ascontiguousarray(w_cache)), b, m, n_feat, _p(grad_out))


def field_eval_model(coords, params, spec: GridSpec, weights, relu_out: bool = True):
    """_kernels.py:154-176 field_eval_model (per-sample serial fp32; == eval_fused)."""
    coords = np.ascontiguousarray(coords, dtype=np.float32)
    res, entries, dense, off = level_tables(spec)
    flat = np.concatenate([np.asarray(w, dtype=np.float32).ravel() for w in weights])
    widths = np.array([weights[0].shape[1]] + [w.shape[0] for w in weights], dtype=np.int32)
    out = np.empty(coords.shape[0], dtype=np.float32)
    lib().orc_field_eval_model(_p(coords), coords.shape[0], _p(np.ascontiguousarray(params, np.float32)),
                               _p(off), _p(res), _p(entries), _p(dense), spec.n_levels,
                               spec.n_features_per_level, _p(flat), _p(widths), len(weights),
                               int(bool(relu_out)), _p(out))
    return out


# ---------------------------------------------------------------- MLP + loss (numpy, as the reference)

def mlp_forward(x, weights, relu_out: bool = True):
    """network.py:61-74: h = relu(h @ W.T) per layer (output ReLU if relu_out)."""
    acts = [x]
    h = x
    last = len(weights) - 1
    for i, w in enumerate(weights):
        h = h @ w.T
        if i < last or relu_out:
            h = np.maximum(h, 0)
        acts.append(h)
    return h[:, 0], acts


def mlp_backward(acts, weights, grads, dl_dout, relu_out: bool = True):
    """network.py:76-93: accumulate dW_i, return dL/dinput."""
    d = np.asarray(dl_dout, dtype=weights[0].dtype)[:, None]
    last = len(weights) - 1
    for i in range(last, -1, -1):
        if i < last or relu_out:
            d = d * (acts[i + 1] > 0)
        grads[i] += d.T @ acts[i]
        if i > 0:
            d = d @ weights[i]
    return d @ weights[0]


def loss_and_grad(pred, target, kind: str = "L1"):
    """network.py:96-114 (f64 reduction, grad cast to pred dtype)."""
    b = pred.shape[0]
    diff = pred.astype(np.float64) - target.astype(np.float64)
    if kind == "L1":
        loss = float(np.mean(np.abs(diff)))
        grad = np.sign(diff) / b
    else:
        loss = float(np.mean(diff * diff))
        grad = 2.0 * diff / b
    return loss, grad.astype(pred.dtype)


# ---------------------------------------------------------------- optimizer

@dataclass
class AdamState:
    """network.py:117-130 OptimizerState defaults."""
    base_lr: float = 0.005
    beta1: float = 0.9
    beta2: float = 0.999
    epsilon: float = 1e-15
    l2_reg: float = 1e-6
    decay_start: int = 2000
    decay_interval: int = 1000
    decay_base: float = 0.99
    t: int = 0
    m: list = field(default_factory=list)
    v: list = field(default_factory=list)


def lr_at(opt: AdamState, t: int) -> float:
    """network.py:153-157."""
    return opt.base_lr * opt.decay_base ** (max(0, t - opt.decay_start) // opt.decay_interval)


def adam_scalars(opt: AdamState):
    """network.py:163-181: the float32-cast scalars of one Adam step."""
    f = np.float32
    step = opt.t + 1
    c1 = 1.0 - opt.beta1 ** step
    c2 = 1.0 - opt.beta2 ** step
    return (f(lr_at(opt, opt.t)), f(opt.beta1), f(1.0 - opt.beta1), f(opt.beta2), f(1.0 - opt.beta2),
            f(c1), f(c2), f(opt.epsilon), f(opt.l2_reg))


def adam_step(opt: AdamState, params, grads) -> None:
    """network.py:160-183 for float32 groups (restated in C, bit-identical)."""
    if not opt.m:
        opt.m = [np.zeros_like(p) for p in params]
        opt.v = [np.zeros_like(p) for p in params]
    sc = adam_scalars(opt)
    for gi, (p, g) in enumerate(zip(params, grads)):
        bad = np.isnan(g)
        if bad.any():
            j = int(np.flatnonzero(bad.ravel())[0])
            raise FloatingPointError(f"NaN gradient in parameter group {gi} at flat index {j}")
        lib().orc_adam_f32(_p(p), _p(g), _p(opt.m[gi]), _p(opt.v[gi]), p.size,
                           sc[0], sc[1], sc[2], sc[3], sc[4], sc[5], sc[6], sc[7], sc[8])
    opt.t += 1


# ---------------------------------------------------------------- random stream + GT lookup

def pcg64_initial_state(seed: int):
    """numpy.random.default_rng(seed).bit_generator.state (numpy 2.3.5) as (state, inc)."""
    st = np.random.default_rng(seed).bit_generator.state["state"]
    return int(st["state"]), int(st["inc"])


def pcg64_random_f32(seed_or_state, u32_offset: int, count: int) -> np.ndarray:
    """float32 draws u32_offset..u32_offset+count of default_rng(seed).random(dtype=float32)."""
    if isinstance(seed_or_state, tuple):
        s, inc = seed_or_state
    else:
        s, inc = pcg64_initial_state(int(seed_or_state))
    out = np.empty(count, dtype=np.float32)
    m64 = (1 << 64) - 1
    lib().orc_pcg64_random_f32(s >> 64, s & m64, inc >> 64, inc & m64, int(u32_offset), count, _p(out))
    return out


def trilinear(norm: np.ndarray, pts: np.ndarray, clip: bool = False) -> np.ndarray:
    """volume.py:148-164 _gather_corners on a (dz,dy,dx) float32 normalised array."""
    norm = np.ascontiguousarray(norm, dtype=np.float32)
    pts = np.ascontiguousarray(pts, dtype=np.float32)
    dz, dy, dx = norm.shape
    out = np.empty(pts.shape[0], dtype=np.float32)
    lib().orc_trilinear(_p(norm), dx, dy, dz, _p(pts), pts.shape[0], int(clip), _p(out))
    return out


class InCoreSampler:
    """sampler.py:263-270 + 64-74: uniform f32 coords from default_rng(seed), trilinear targets."""

    def __init__(self, norm: np.ndarray, seed: int = 0):
        self.norm = np.ascontiguousarray(norm, dtype=np.float32)
        self.state = pcg64_initial_state(seed)
        self.u32 = 0

    def sample(self, b: int):
        coords = pcg64_random_f32(self.state, self.u32, 3 * b).reshape(b, 3)
        self.u32 += 3 * b
        return coords, trilinear(self.norm, coords, clip=True)


# ---------------------------------------------------------------- analytic fields (fields.py:15-88)

def _gauss(p, center, sigma):
    d2 = np.sum((p - np.asarray(center, dtype=p.dtype)) ** 2, axis=-1)
    return np.exp(-d2 / (2.0 * sigma * sigma))


def field_fn(name: str):
    def gauss(p):
        return _gauss(p, (0.5, 0.5, 0.5), 0.18)

    def blobs(p):
        return np.maximum(np.maximum(_gauss(p, (0.30, 0.32, 0.28), 0.09),
                                     _gauss(p, (0.68, 0.60, 0.55), 0.07)),
                          _gauss(p, (0.45, 0.75, 0.72), 0.06))

    def waves(p):
        x, y, z = p[..., 0], p[..., 1], p[..., 2]
        return 0.5 + 0.5 * (np.sin(2.0 * np.pi * 3 * x) * np.sin(2.0 * np.pi * 2 * y)
                            * np.sin(2.0 * np.pi * 4 * z))

    def mlobb(p):
        fm, alpha = 6.0, 0.25
        q = 2.0 * np.asarray(p, dtype=np.float64) - 1.0
        x, y, z = q[..., 0], q[..., 1], q[..., 2]
        r = np.sqrt(x * x + y * y)
        rho = np.cos(2.0 * np.pi * fm * 0.5 * np.cos(np.pi * r / 2.0))
        v = (1.0 - np.sin(np.pi * z / 2.0) + alpha * (1.0 + rho)) / (2.0 * (1.0 + alpha))
        return np.clip(v, 0.0, 1.0)

    return {"gauss": gauss, "blobs": blobs, "waves": waves, "mlobb": mlobb}[name]


def rasterize(name: str, dims) -> np.ndarray:
    """fields.py:67-88 for dtype f32, range (0,1): returns the (dz,dy,dx) normalised array."""
    dx, dy, dz = dims
    zs = (np.arange(dz, dtype=np.float64) + 0.5) / dz
    ys = (np.arange(dy, dtype=np.float64) + 0.5) / dy
    xs = (np.arange(dx, dtype=np.float64) + 0.5) / dx
    gz, gy, gx = np.meshgrid(zs, ys, xs, indexing="ij")
    vals = np.clip(field_fn(name)(np.stack([gx, gy, gz], axis=-1)), 0.0, 1.0)
    return vals.astype(np.float32)


# ---------------------------------------------------------------- model (model.py:95-253)

def net_from_config(cfg: dict):
    """model.py:214-253 subset: (GridSpec, n_neurons, n_hidden, relu_out, loss, batch, opt)."""
    enc = cfg.get("encoding", {})
    otype = enc.get("otype", "HashGrid")
    spec = GridSpec(kind={"HashGrid": "hashgrid", "DenseGrid": "densegrid"}[otype],
                    n_levels=int(enc.get("n_levels", 8)),
                    n_features_per_level=int(enc.get("n_features_per_level", 4)),
                    log2_hashmap_size=int(enc.get("log2_hashmap_size", 15)),
                    base_resolution=int(enc.get("base_resolution", 4)),
                    per_level_scale=float(enc.get("per_level_scale", 2.0)))
    net = cfg.get("network", {})
    relu_out = str(net.get("output_activation", "ReLU")).lower() == "relu"
    opt = AdamState()
    o = cfg.get("optimizer", {})
    if o.get("otype", "ExponentialDecay") == "ExponentialDecay":
        opt.decay_start = int(o.get("decay_start", opt.decay_start))
        opt.decay_interval = int(o.get("decay_interval", opt.decay_interval))
        opt.decay_base = float(o.get("decay_base", opt.decay_base))
        nested = o.get("nested", {})
    else:
        opt.decay_base = 1.0
        nested = o
    opt.base_lr = float(nested.get("learning_rate", opt.base_lr))
    opt.beta1 = float(nested.get("beta1", opt.beta1))
    opt.beta2 = float(nested.get("beta2", opt.beta2))
    opt.epsilon = float(nested.get("epsilon", opt.epsilon))
    opt.l2_reg = float(nested.get("l2_reg", opt.l2_reg))
    return (spec, int(net.get("n_neurons", 64)), int(net.get("n_hidden_layers", 4)), relu_out,
            cfg.get("loss", {}).get("otype", "L1"), int(cfg.get("batch_size", 65536)), opt)


class OracleModel:
    """NeuralModel restated (model.py:95-214) for float32 hash/dense-grid models."""

    def __init__(self, cfg: dict, seed: int = 0):
        (self.spec, nn, nh, self.relu_out, self.loss_kind, self.batch_size, self.opt) = net_from_config(cfg)
        rng = np.random.default_rng(seed)                       # model.py:235
        res, entries, dense, off = level_tables(self.spec)
        total = int((entries * self.spec.n_features_per_level).sum())
        # encoding.py:167-168, then network.py:49-54 from the same generator
        self.params = rng.uniform(-FEATURE_INIT_SCALE, FEATURE_INIT_SCALE, size=total).astype(np.float32)
        self.param_grads = np.zeros(total, dtype=np.float32)
        widths = [self.spec.out_width] + [nn] * nh + [1]
        self.weights = []
        for fan_in, fan_out in zip(widths[:-1], widths[1:]):
            bound = math.sqrt(6.0 / fan_in)
            self.weights.append(rng.uniform(-bound, bound, size=(fan_out, fan_in)).astype(np.float32))
        self.grads = [np.zeros_like(w) for w in self.weights]

    @property
    def n_params(self) -> int:
        return self.params.size + sum(w.size for w in self.weights)

    def flat_params(self) -> np.ndarray:
        """trainer.py:114-123 blob order."""
        return np.concatenate([self.params] + [w.ravel() for w in self.weights])

    def load_flat(self, blob: np.ndarray) -> None:
        k = self.params.size
        self.params[...] = blob[:k]
        pos = k
        for w in self.weights:
            w[...] = blob[pos:pos + w.size].reshape(w.shape)
            pos += w.size

    def encode_batch(self, coords):
        return grid_encode_fwd(coords, self.params, self.spec)

    def train_step(self, coords, targets, capture: dict | None = None) -> float:
        """model.py:154-174: encode -> MLP -> loss -> backprop -> Adam; returns pre-update loss."""
        feats, idx, w = self.encode_batch(coords)
        pred, acts = mlp_forward(feats, self.weights, self.relu_out)
        loss, dl_dpred = loss_and_grad(pred, targets.astype(pred.dtype), self.loss_kind)
        dl_dfeat = mlp_backward(acts, self.weights, self.grads, dl_dpred, self.relu_out)
        grid_encode_bwd(np.ascontiguousarray(dl_dfeat, dtype=np.float32), idx, w,
                        self.spec.n_features_per_level, self.param_grads)
        if capture is not None:
            capture.update(feats=feats, pred=pred, dl_dpred=dl_dpred, dl_dfeat=dl_dfeat,
                           enc_grads=self.param_grads.copy(), w_grads=[g.copy() for g in self.grads])
        adam_step(self.opt, [self.params] + self.weights, [self.param_grads] + self.grads)
        return loss

    def eval_batch(self, coords):
        """model.py:178-182."""
        feats, _, _ = grid_encode_fwd(coords, self.params, self.spec, want_cache=False)
        return mlp_forward(feats, self.weights, self.relu_out)[0].astype(np.float32)

    def eval_fused(self, coords):
        """model.py:184-198."""
        return field_eval_model(coords, self.params, self.spec, self.weights, self.relu_out)


def decode(model: OracleModel, dims, value_range=(0.0, 1.0), slab_z: int = 16, fused: bool = False):
    """trainer.py:80-106 decode_slabs + decode -> (dz,dy,dx) float32."""
    dx, dy, dz = dims
    lo, hi = value_range
    xs = (np.arange(dx, dtype=np.float32) + np.float32(0.5)) / np.float32(dx)
    ys = (np.arange(dy, dtype=np.float32) + np.float32(0.5)) / np.float32(dy)
    out = np.empty((dz, dy, dx), dtype=np.float32)
    for z0 in range(0, dz, slab_z):
        nz = min(slab_z, dz - z0)
        zs = (np.arange(z0, z0 + nz, dtype=np.float32) + np.float32(0.5)) / np.float32(dz)
        gz, gy, gx = np.meshgrid(zs, ys, xs, indexing="ij")
        coords = np.stack([gx.ravel(), gy.ravel(), gz.ravel()], axis=1)
        vals = (model.eval_fused(coords) if fused else model.eval_batch(coords)).astype(np.float64)
        out[z0:z0 + nz] = (vals * (hi - lo) + lo).astype(np.float32).reshape(nz, dy, dx)
    return out


def psnr(a: np.ndarray, b: np.ndarray) -> float:
    """volume.py:197-207 on already-normalised arrays."""
    d = a.astype(np.float64) - b.astype(np.float64)
    e = float(np.mean(d * d))
    return 99.0 if e == 0.0 else -10.0 * math.log10(e)
