"""Volume renderers over a field (neural model or dense grid) on the B200.

Mirror of the reference's render.py (/root/reference/pkg/src/neuralvol/
render.py): RenderConfig, FrameStats, Framebuffer, accumulate,
ensure_macrocells, render_reference (in-shader: one thread per ray, Phi
inline), render_wavefront (sample streaming: stage K samples per ray, one
batched Phi evaluation, shade, compact) and render.  Both architectures run
in csrc/render.cu behind nvol_render.  The path-tracing mode of the
reference (render.py:361-368, 396-423) is outside this build's hot path and
raises ConfigError.
"""
from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .camera import Camera
from .errors import ConfigError
from .macrocell import MacroCellGrid, macrocell_build, macrocell_from_model, macrocell_set_tf
from .model import NeuralModel
from .transfer import TransferFunction, tf_max_opacity
from .volume import ScalarField

MODES = ("raymarch", "raymarch_shadow", "pathtrace")
TERMINATION = 1e-3  # render.py:28


def _unit3(v, what: str):
    a = np.asarray(v, dtype=np.float64)
    if a.shape != (3,) or not np.all(np.isfinite(a)):
        raise ConfigError(f"{what} must be three finite components, got {v!r}")
    n = float(np.linalg.norm(a))
    if n == 0.0:
        raise ConfigError(f"{what} must be nonzero")
    return tuple(a / n)


@dataclass
class RenderConfig:
    """render.py:41-94."""
    mode: str = "raymarch"
    use_macrocells: bool = False
    frames: int = 1
    step_size: float = 1.0
    max_step: float = 64.0
    step_exponent: float = 2.0
    rr_depth: int = 4
    k_batch: int = 8
    light_direction: tuple = (-0.57735026919, -0.57735026919, -0.57735026919)
    light_radiance: tuple = (1.0, 1.0, 1.0)
    background: tuple = (1.0, 1.0, 1.0)
    seed: int = 0
    ambient: float = 0.2
    skip_empty: bool = True

    def __post_init__(self) -> None:
        if self.mode not in MODES:
            raise ConfigError(f"unknown render mode {self.mode!r}; expected one of {MODES}")
        if not self.step_size > 0:
            raise ConfigError(f"step_size must be > 0, got {self.step_size}")
        if self.max_step < self.step_size:
            raise ConfigError(f"max_step {self.max_step} < step_size {self.step_size}")
        if self.k_batch < 1:
            raise ConfigError(f"k_batch must be >= 1, got {self.k_batch}")
        if self.frames < 1:
            raise ConfigError(f"frames must be >= 1, got {self.frames}")
        if self.rr_depth < 0:
            raise ConfigError(f"rr_depth must be >= 0, got {self.rr_depth}")
        if not 0.0 <= self.ambient <= 1.0:
            raise ConfigError(f"ambient must be in [0,1], got {self.ambient}")
        self.light_direction = _unit3(self.light_direction, "light direction")
        self.light_radiance = tuple(float(c) for c in self.light_radiance)
        self.background = tuple(float(c) for c in self.background)
        if len(self.light_radiance) != 3 or len(self.background) != 3:
            raise ConfigError("light radiance and background must have three components")

    def to_json(self) -> dict:
        return {"mode": self.mode, "use_macrocells": self.use_macrocells, "frames": self.frames,
                "step_size": self.step_size, "max_step": self.max_step, "step_exponent": self.step_exponent,
                "rr_depth": self.rr_depth, "k_batch": self.k_batch,
                "light": {"direction": list(self.light_direction), "radiance": list(self.light_radiance)},
                "background": list(self.background), "seed": self.seed, "ambient": self.ambient,
                "skip_empty": self.skip_empty}


def render_config_from_json(obj: dict) -> RenderConfig:
    """render.py:97-128."""
    if not isinstance(obj, dict):
        raise ConfigError(f"render config must be an object, got {type(obj).__name__}")
    light = obj.get("light", {})
    kw = {}

    def take(name, *aliases, convert=None):
        for key in (name,) + aliases:
            if key in obj:
                kw[name] = convert(obj[key]) if convert else obj[key]
                return

    take("mode", convert=str)
    take("use_macrocells", "macrocells", convert=bool)
    take("frames", "spp", convert=int)
    take("step_size", convert=float)
    take("max_step", convert=float)
    take("step_exponent", convert=float)
    take("rr_depth", convert=int)
    take("k_batch", "k", convert=int)
    take("background", convert=tuple)
    take("seed", convert=int)
    take("ambient", convert=float)
    take("skip_empty", convert=bool)
    if "direction" in light:
        kw["light_direction"] = tuple(light["direction"])
    if "radiance" in light:
        kw["light_radiance"] = tuple(light["radiance"])
    try:
        return RenderConfig(**kw)
    except TypeError as e:
        raise ConfigError(f"bad render config: {e}") from None


@dataclass
class FrameStats:
    """render.py:131-144."""
    evals: int = 0
    violations: int = 0
    alive_per_iteration: list = field(default_factory=list)
    ms: float = 0.0

    def to_json(self) -> dict:
        return {"field_evaluations": self.evals, "majorant_violations": self.violations,
                "rays_alive_per_iteration": list(self.alive_per_iteration), "ms": self.ms}


@dataclass
class Framebuffer:
    """Running mean of frames in float64 (render.py:147-172), on the device."""
    width: int
    height: int
    total: object = None
    count: int = 0

    def __post_init__(self) -> None:
        if self.total is None:
            self.total = torch.zeros((self.height, self.width, 3), dtype=torch.float64, device=_lib.device())

    def reset(self) -> None:
        self.total.zero_()
        self.count = 0

    @property
    def mean(self) -> torch.Tensor:
        if self.count == 0:
            return torch.zeros_like(self.total)
        return self.total / self.count

    def to_u8(self) -> np.ndarray:
        m = torch.clamp(self.mean, 0.0, 1.0)
        return torch.floor(m * 255.0 + 0.5).to(torch.uint8).cpu().numpy()


def accumulate(fb: Framebuffer, frame, n: int | None = None):
    """render.py:175-183."""
    f = frame if isinstance(frame, torch.Tensor) else torch.as_tensor(np.asarray(frame))
    if tuple(f.shape) != tuple(fb.total.shape):
        raise ConfigError(f"frame shape {tuple(f.shape)} != framebuffer {tuple(fb.total.shape)}")
    fb.total += f.to(fb.total.device, torch.float64)
    fb.count += 1
    if n is not None and n != fb.count:
        raise ConfigError(f"accumulation count mismatch: caller says {n}, buffer has {fb.count}")
    return fb.mean


def ensure_macrocells(phi, tf: TransferFunction, cfg: RenderConfig, grid: MacroCellGrid | None):
    """render.py:246-257."""
    if not cfg.use_macrocells:
        return None
    if grid is None:
        grid = macrocell_build(phi) if isinstance(phi, ScalarField) else macrocell_from_model(phi)
    macrocell_set_tf(grid, tf)
    return grid


_WS: dict = {}


def _workspace(npix: int, k: int) -> torch.Tensor:
    need = int(_lib.load().nvol_render_workspace_bytes(npix, k))
    key = (npix, k)
    if key not in _WS or _WS[key].numel() < need:
        _WS.clear()
        _WS[key] = torch.empty(need, dtype=torch.uint8, device=_lib.device())
    return _WS[key]


def render_frame_device(phi, tf: TransferFunction, cam: Camera, cfg: RenderConfig, grid: MacroCellGrid | None,
                        architecture: str = "wavefront", eval_mode: str | None = None, rows=None, frame: int = 0):
    """One frame on the device -> (image (H,W,3) float32 device tensor, FrameStats).

    rows=(row0, nrows) renders only that image tile (an (nrows,W,3) image):
    rays are independent, so tiles of a frame assemble bit-identically
    (the multi-GPU split, distributed.render_tile)."""
    row0, nrows = (0, cam.height) if rows is None else (int(rows[0]), int(rows[1]))
    if row0 < 0 or nrows < 1 or row0 + nrows > cam.height:
        raise ConfigError(f"bad image tile rows {rows} for height {cam.height}")
    if architecture not in ("wavefront", "reference"):
        raise ConfigError(f"unknown architecture {architecture!r}; expected one of ['reference', 'wavefront']")
    dev = _lib.device()
    if isinstance(phi, ScalarField):
        dims = phi.meta.dims
        norm = phi.normalized
        field_args = (1, _lib.ptr(norm), norm.shape[2], norm.shape[1], norm.shape[0], None, None, None, None, None,
                      1, 1, None, None, 1, 0)
        emode = 0
        img_ptr_keep = norm
    elif isinstance(phi, NeuralModel):
        if not phi._use_kernels():
            raise ConfigError("renderers require a float32 grid-encoded model; "
                              f"got encoder {type(phi.encoder).__name__}, dtype {np.dtype(phi.dtype).name}")
        dims = phi.dims
        c = phi.encoder.config
        off, res, ent, dense = phi.encoder.c_tables()
        widths = phi._widths()
        field_args = (0, None, 1, 1, 1, _lib.ptr(phi.flat_params), off, res, ent, dense, c.n_levels,
                      c.n_features_per_level, _lib.ptr(phi._weights_flat()), _lib.host_i32(widths), len(widths) - 1,
                      int(phi.mlp.config.output_activation == "relu"))
        emode = 1 if (eval_mode or phi.infer_mode) == "tensor" else 0
        img_ptr_keep = None
    else:
        raise ConfigError(f"cannot render a {type(phi).__name__}; expected ScalarField or NeuralModel")
    if cfg.use_macrocells:
        if grid is None:
            raise ConfigError("macro-cell rendering needs a grid; call ensure_macrocells")
        if tuple(grid.vol_dims) != tuple(dims):
            raise ConfigError(f"macro-cell grid dims {grid.vol_dims} != field dims {tuple(dims)}")
        mu, ng = grid.mu_max, float(grid.n_g)
    else:
        mu, ng = torch.zeros((1, 1, 1), dtype=torch.float32, device=dev), 1.0
    gz, gy, gx = mu.shape
    cv, crgb, ov, oa = tf.tables
    ld = cfg.light_direction
    seed = int(cfg.seed) & 0xFFFFFFFFFFFFFFFF
    rp = np.array([float(cfg.mode == "raymarch_shadow"), float(cfg.use_macrocells), float(cfg.skip_empty),
                   float(cfg.k_batch), float(np.float32(cfg.step_size)), float(np.float32(cfg.max_step)),
                   float(np.float32(cfg.step_exponent)), float(np.float32(TERMINATION)),
                   float(np.float32(cfg.ambient)), float(np.float32(tf.density_scale)), ng,
                   float(np.float32(-ld[0])), float(np.float32(-ld[1])), float(np.float32(-ld[2])),
                   *[float(np.float32(b)) for b in cfg.background], *[float(d) for d in dims],
                   # path tracing (render.py:291-304 _Scene): seed split in 32-bit halves (exact in f64),
                   # frame, Russian-roulette depth, light radiance (f32), global majorant rounded through f32
                   float(cfg.mode == "pathtrace"), float(seed & 0xFFFFFFFF), float(seed >> 32), float(frame),
                   float(cfg.rr_depth), *[float(np.float32(c)) for c in cfg.light_radiance],
                   float(np.float32(tf_max_opacity(tf, 0.0, 1.0) * tf.density_scale))], dtype=np.float64)
    cp = cam.device_params(row0, nrows)
    npix = cam.width * nrows
    img = torch.empty((nrows, cam.width, 3), dtype=torch.float32, device=dev)
    ws = _workspace(npix, cfg.k_batch)
    stats = (ctypes_i64 := np.zeros(3, dtype=np.int64))
    hist = np.zeros(4096, dtype=np.int32)
    mlp_img = phi.mlp_image() if (isinstance(phi, NeuralModel) and emode == 1) else None
    c64 = np.ctypeslib.as_ctypes
    t0 = time.perf_counter()
    _lib.call("nvol_render", c64(cp), c64(rp), c64(np.ascontiguousarray(cv)), c64(np.ascontiguousarray(crgb).ravel()),
              len(cv), c64(np.ascontiguousarray(ov)), c64(np.ascontiguousarray(oa)), len(ov), _lib.ptr(mu), gx, gy,
              gz, *field_args, 0 if architecture == "wavefront" else 1, emode, _lib.ptr(mlp_img), _lib.ptr(img),
              _lib.ptr(ws), ws.numel(), c64(ctypes_i64), c64(hist), len(hist), _lib.stream())
    ms = (time.perf_counter() - t0) * 1e3
    del img_ptr_keep
    iters = int(stats[1])
    return img, FrameStats(evals=int(stats[0]), violations=int(stats[2]),
                           alive_per_iteration=hist[:min(iters, len(hist))].tolist(),
                           ms=ms)


def _one(architecture):
    def run(phi, tf, cam, cfg, grid=None, frame: int = 0, stats_out: list | None = None):
        if cfg.use_macrocells and grid is None:
            grid = ensure_macrocells(phi, tf, cfg, None)
        img, st = render_frame_device(phi, tf, cam, cfg, grid, architecture, frame=frame)
        if stats_out is not None:
            stats_out.append(st)
        return img.cpu().numpy()
    return run


render_reference = _one("reference")
render_reference.__doc__ = "In-shader renderer: one thread per ray to completion (render.py:347-380)."
render_wavefront = _one("wavefront")
render_wavefront.__doc__ = "Sample-streaming renderer: stage, batch-infer, shade, compact (render.py:383-454)."


def render(phi, tf: TransferFunction, cam: Camera, cfg: RenderConfig, architecture: str = "wavefront",
           grid: MacroCellGrid | None = None, stats_out: list | None = None, device_output: bool = False):
    """Accumulate cfg.frames frames and return the running mean (H,W,3) float32 (render.py:460-475)."""
    if architecture not in ("reference", "wavefront"):
        raise ConfigError(f"unknown architecture {architecture!r}; expected one of ['reference', 'wavefront']")
    grid = ensure_macrocells(phi, tf, cfg, grid)
    fb = Framebuffer(cam.width, cam.height)
    for f in range(cfg.frames):
        img, st = render_frame_device(phi, tf, cam, cfg, grid, architecture, frame=f)
        if stats_out is not None:
            stats_out.append(st)
        accumulate(fb, img)
    m = fb.mean.to(torch.float32)
    return m if device_output else m.cpu().numpy()
