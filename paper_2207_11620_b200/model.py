"""NeuralModel: encoder + MLP + optimizer + loss, the representation Phi.

Mirror of the reference's model.py (/root/reference/pkg/src/neuralvol/
model.py:95-253): same tcnn-style JSON config handling, same initialisation
stream, same method surface (encode_batch, train_step, eval_batch,
eval_fused, param_groups, config_json, build_model).

B200 layout: all trainable parameters live in ONE flat device buffer
[encoder table | pad to 16 B | W_0 | W_1 | ...] with identically laid-out
gradient and Adam-moment buffers.  `encoder.params`, `mlp.weights[i]`,
`opt.m[i]` ... are views into those buffers, so the reference's per-group API
keeps working while the training step runs as a few large kernels over the
flat buffers (one Adam launch, one all-reduce for data parallelism).
"""
from __future__ import annotations

import os

from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch

from . import _lib
from ._tensor import out, to_device, torch_dtype
from .encoding import EncoderConfig, GridEncoder, make_encoder
from .errors import ConfigError
from .network import Mlp, MlpConfig, OptimizerState, adam_scalars, adam_step, loss_and_grad

_ENCODER_OTYPES = {
    "Identity": "identity",
    "Frequency": "frequency",
    "OneBlob": "oneblob",
    "DenseGrid": "densegrid",
    "HashGrid": "hashgrid",
}
_ENCODER_KIND_TO_OTYPE = {v: k for k, v in _ENCODER_OTYPES.items()}

# Training-step engines (nvol_train_fwd_bwd `mode`).
NAN_NONE = (1 << 63) - 1   # nvol.h NaN contract: no parameter group holds a NaN gradient
MODE_SIMT = 0      # generic kernels, fp32 CUDA cores
MODE_TCGEN05 = 1   # fused tile pipeline, tcgen05 fp16 operands / fp32 accumulate
TRAIN_PREENCODED = 16   # mode flag, nvol.h NVOL_TRAIN_PREENCODED
TRAIN_ENCODE_ONLY = 32  # mode flag, nvol.h NVOL_TRAIN_ENCODE_ONLY


def encoder_config_from_json(obj: dict) -> EncoderConfig:
    """model.py:31-45."""
    otype = obj.get("otype", "HashGrid")
    if otype not in _ENCODER_OTYPES:
        raise ConfigError(f"unknown encoding otype {otype!r}; expected one of {sorted(_ENCODER_OTYPES)}")
    defaults = EncoderConfig(kind=_ENCODER_OTYPES[otype])
    return EncoderConfig(
        kind=defaults.kind,
        n_levels=int(obj.get("n_levels", defaults.n_levels)),
        n_features_per_level=int(obj.get("n_features_per_level", defaults.n_features_per_level)),
        log2_hashmap_size=int(obj.get("log2_hashmap_size", defaults.log2_hashmap_size)),
        base_resolution=int(obj.get("base_resolution", defaults.base_resolution)),
        per_level_scale=float(obj.get("per_level_scale", defaults.per_level_scale)),
        n_frequencies=int(obj.get("n_frequencies", defaults.n_frequencies)),
        n_bins=int(obj.get("n_bins", defaults.n_bins)),
    )


def encoder_config_to_json(cfg: EncoderConfig) -> dict:
    """model.py:48-62."""
    o = {"otype": _ENCODER_KIND_TO_OTYPE[cfg.kind]}
    if cfg.kind in ("densegrid", "hashgrid"):
        o.update(n_levels=cfg.n_levels, n_features_per_level=cfg.n_features_per_level,
                 log2_hashmap_size=cfg.log2_hashmap_size, base_resolution=cfg.base_resolution,
                 per_level_scale=cfg.per_level_scale)
    elif cfg.kind == "frequency":
        o["n_frequencies"] = cfg.n_frequencies
    elif cfg.kind == "oneblob":
        o["n_bins"] = cfg.n_bins
    return o


def optimizer_from_json(obj: dict) -> OptimizerState:
    """model.py:65-83."""
    opt = OptimizerState()
    if obj.get("otype", "ExponentialDecay") == "ExponentialDecay":
        opt.decay_start = int(obj.get("decay_start", opt.decay_start))
        opt.decay_interval = int(obj.get("decay_interval", opt.decay_interval))
        opt.decay_base = float(obj.get("decay_base", opt.decay_base))
        nested = obj.get("nested", {})
    else:
        opt.decay_base = 1.0
        nested = obj
    if nested.get("otype", "Adam") != "Adam":
        raise ConfigError(f"unsupported optimizer otype {nested.get('otype')!r}")
    opt.base_lr = float(nested.get("learning_rate", opt.base_lr))
    opt.beta1 = float(nested.get("beta1", opt.beta1))
    opt.beta2 = float(nested.get("beta2", opt.beta2))
    opt.epsilon = float(nested.get("epsilon", opt.epsilon))
    opt.l2_reg = float(nested.get("l2_reg", opt.l2_reg))
    return opt


def default_config() -> dict:
    """model.py:86-92."""
    return {
        "loss": {"otype": "L1"},
        "optimizer": OptimizerState().to_json(),
        "encoding": encoder_config_to_json(EncoderConfig()),
        "network": {"otype": "MLP", "n_neurons": 64, "n_hidden_layers": 4, "output_activation": "ReLU"},
    }


@dataclass
class NeuralModel:
    """model.py:95-214, backed by flat device buffers (module docstring)."""
    encoder: GridEncoder
    mlp: Mlp
    opt: OptimizerState
    loss_kind: str = "L1"
    batch_size: int = 65536
    value_range: tuple = (0.0, 1.0)
    dims: tuple = (2, 2, 2)

    def __post_init__(self) -> None:
        if self.encoder.out_width != self.mlp.config.input_width:
            raise ConfigError(
                f"encoder width {self.encoder.out_width} != MLP input width {self.mlp.config.input_width}")
        if self.batch_size < 1:
            raise ConfigError("batch_size must be >= 1")
        if self.loss_kind not in ("L1", "L2"):
            raise ConfigError(f"unknown loss otype {self.loss_kind!r}; expected 'L1' or 'L2'")
        self.train_mode = MODE_SIMT
        self.infer_mode = "exact"        # eval_fused / eval_batch / decode: "exact" or "tensor"
        self._pack()
        self._ws = None
        self._stage = None
        # training engine: the tcgen05 pipeline wherever the device and the shape take it
        # (north-star parity bar for half-precision operands: 1e-2; PSNR within 0.1 dB,
        # test_psnr_ensemble_within_0p1_db), else the fp32 SIMT engine.  NVOL_TRAIN_ENGINE=simt
        # (or train_mode = MODE_SIMT) selects the fp32 engine; deterministic mode always does.
        if os.environ.get("NVOL_TRAIN_ENGINE", "auto") != "simt" and self._tc_device():
            self.train_mode = MODE_TCGEN05

    # ---------------------------------------------------------------- flat buffers
    def _pack(self) -> None:
        dt = torch_dtype(self.mlp.dtype)
        dev = self.encoder.params.device
        k = self.encoder.n_params
        self.enc_size = k
        # front pad (floats) so that the hashed levels' entry pairs {2j, 2j+1} are 16-byte
        # aligned (one float4 gather / RED per x-adjacent corner pair); every flat buffer is
        # a view `lead` floats into a 16-byte-aligned allocation (nvol.h flat layout)
        enc = self.encoder
        hashed = [int(o) for o, d in zip(getattr(enc, "level_offsets", []), getattr(enc, "_dense", [])) if not d]
        lead = (-hashed[0]) % 4 if (hashed and dt == torch.float32) else 0
        if os.environ.get("NVOL_FLAT_LEAD") is not None:   # layout experiments
            lead = int(os.environ["NVOL_FLAT_LEAD"]) % 4
        self.flat_lead = lead
        self.w_offset = ((lead + k + 3) & ~3) - lead   # 16-byte aligned weights (tcgen05 staging)
        self.w_shapes = [tuple(w.shape) for w in self.mlp.weights]
        total = self.w_offset + sum(int(np.prod(s)) for s in self.w_shapes)
        self.flat_size = ((lead + total + 3) & ~3) - lead

        def alloc():
            return torch.zeros(lead + self.flat_size, dtype=dt, device=dev)[lead:]
        self.flat_params = alloc()
        self.flat_grads = alloc()
        self.flat_m = alloc()
        self.flat_v = alloc()
        self.flat_params[:k].copy_(self.encoder.params)
        pos = self.w_offset
        for w in self.mlp.weights:
            self.flat_params[pos:pos + w.numel()].copy_(w.reshape(-1))
            pos += w.numel()
        self._bind_views()

    def rehome_flat(self, capacity: int) -> None:
        """Move the four flat buffers into allocations holding `capacity` >= flat_size
        floats (zero padding after the model), keeping the lead pad, so collectives can
        work on equal-sized chunks of `flat_*_padded`; re-binds every view.  Existing
        CUDA graphs / pipelines that captured the old pointers must be rebuilt."""
        capacity = int(capacity)
        if capacity < self.flat_size:
            raise ConfigError(f"capacity {capacity} < flat size {self.flat_size}")
        lead = self.flat_lead
        for name in ("flat_params", "flat_grads", "flat_m", "flat_v"):
            old = getattr(self, name)
            buf = torch.zeros(lead + capacity, dtype=old.dtype, device=old.device)[lead:]
            buf[:self.flat_size].copy_(old)
            setattr(self, name + "_padded", buf)
            setattr(self, name, buf[:self.flat_size])
        self._bind_views()
        self._pipeline = None

    def _views(self, flat: torch.Tensor):
        enc = flat[:self.enc_size]
        ws, pos = [], self.w_offset
        for s in self.w_shapes:
            n = int(np.prod(s))
            ws.append(flat[pos:pos + n].view(*s))
            pos += n
        return enc, ws

    def _bind_views(self) -> None:
        self.encoder.params, self.mlp.weights = self._views(self.flat_params)
        self.encoder.param_grads, self.mlp.grads = self._views(self.flat_grads)
        em, wm = self._views(self.flat_m)
        ev, wv = self._views(self.flat_v)
        self.opt.m, self.opt.v = [em] + wm, [ev] + wv

    # ---------------------------------------------------------------- params
    @property
    def n_params(self) -> int:
        return self.encoder.n_params + self.mlp.n_params

    def param_groups(self):
        return [self.encoder.params] + self.mlp.weights, [self.encoder.param_grads] + self.mlp.grads

    @property
    def dtype(self) -> np.dtype:
        return self.mlp.dtype

    def blob(self) -> torch.Tensor:
        """Parameters in .vnr blob order (trainer.py:114-123), on the device."""
        enc, ws = self._views(self.flat_params)
        return torch.cat([enc] + [w.reshape(-1) for w in ws])

    def load_blob(self, blob) -> None:
        t, _ = to_device(blob, self.mlp.dtype)
        k = self.enc_size
        self.flat_params[:k].copy_(t[:k])
        self.flat_params[self.w_offset:self.w_offset + t.numel() - k].copy_(t[k:])

    # ---------------------------------------------------------------- fast encode
    def _grid_tables(self):
        """model.py:128-131."""
        enc = self.encoder
        res, entries, dense, offsets = enc.kernel_tables()
        return enc.params, offsets, res, entries, dense

    def _use_kernels(self) -> bool:
        """model.py:133-134: the fused fast path is float32 grid models."""
        return isinstance(self.encoder, GridEncoder) and self.dtype == np.float32

    def encode_batch(self, coords):
        """(features, (idx_cache, w_cache)) — model.py:136-150."""
        t, host = to_device(coords, self.dtype)
        feats, idx, w = self.encoder.encode_device(t, want_cache=True, check_nan=False)
        if host:
            return feats.cpu().numpy(), (idx.cpu().numpy(), w.cpu().numpy())
        return feats, (idx, w)

    # ---------------------------------------------------------------- training
    def _widths(self):
        return [self.encoder.out_width] + [self.mlp.config.n_neurons] * self.mlp.config.n_hidden_layers + [1]

    def _workspace(self, b: int) -> torch.Tensor:
        c = self.encoder.config
        need = int(_lib.load().nvol_train_workspace_bytes(b, c.n_levels, c.n_features_per_level,
                                                           self.mlp.config.n_neurons,
                                                           self.mlp.config.n_hidden_layers, self._engine()))
        if self._ws is None or self._ws.numel() < need:
            self._ws = torch.empty(max(need, 256), dtype=torch.uint8, device=self.flat_params.device)
        return self._ws

    def fwd_bwd_device(self, coords: torch.Tensor, targets: torch.Tensor, loss_sum: torch.Tensor,
                       b_global: Optional[int] = None, flags: int = 0,
                       nan_state: Optional[torch.Tensor] = None) -> None:
        """Encode -> MLP -> loss -> backprop -> encoder scatter into flat_grads (no Adam).
        flags (tcgen05 engine): TRAIN_PREENCODED skips the encode (the tile buffer was
        filled by nvol_adam_encode_step), TRAIN_ENCODE_ONLY stops after it.  nan_state
        (int64[2], nvol.h "NaN contract"): NaN-gradient detection and halt."""
        b = coords.shape[0]
        c = self.encoder.config
        ws = self._workspace(b)
        off, res, ent, dense = self.encoder.c_tables()
        _lib.call("nvol_train_fwd_bwd", _lib.ptr(coords), _lib.ptr(targets), b, b_global or b,
                  _lib.ptr(self.flat_params), _lib.ptr(self.flat_grads), off, res, ent, dense, c.n_levels,
                  c.n_features_per_level, self.mlp.config.n_neurons, self.mlp.config.n_hidden_layers,
                  int(self.mlp.config.output_activation == "relu"), 0 if self.loss_kind == "L1" else 1,
                  _lib.ptr(loss_sum), _lib.ptr(ws), ws.numel(), self._engine() | flags, _lib.ptr(nan_state),
                  _lib.stream())

    def _tc_device(self) -> bool:
        try:
            dev = self.flat_params.device
            return bool(dev.type == "cuda" and self.tcgen05_supported()
                        and _lib.load().nvol_has_tcgen05(dev.index or 0))
        except (OSError, RuntimeError):
            return False

    def tcgen05_supported(self) -> bool:
        """Whether the tcgen05 training engine (MODE_TCGEN05) takes this model's shape."""
        c = self.encoder.config
        return bool(self._use_kernels() and _lib.load().nvol_train_tc_supported(
            c.n_levels, c.n_features_per_level, self.mlp.config.n_neurons, self.mlp.config.n_hidden_layers))

    def _engine(self) -> int:
        """Training engine for nvol_train_fwd_bwd: the fp32 SIMT engine (ordered
        reductions) when bitwise repeatability is requested, else train_mode."""
        from .encoding import deterministic
        return MODE_SIMT if deterministic() else self.train_mode

    # ---------------------------------------------------------------- NaN contract
    def group_starts(self) -> list:
        """Flat-buffer start of each parameter group [enc.params, W_0, W_1, ...] (param_groups order)."""
        starts, pos = [0], self.w_offset
        for sh in self.w_shapes:
            starts.append(pos)
            pos += int(np.prod(sh))
        return starts

    def nan_error(self, limit: int) -> FloatingPointError:
        """network.py:167-171: FloatingPointError(group, flat index of the group's first NaN) for the
        NaN state's limit (the start of the first group whose gradient holds a NaN)."""
        starts = self.group_starts()
        gi = max(i for i, st in enumerate(starts) if st <= limit)
        g = self.param_groups()[1][gi].reshape(-1)
        first = torch.empty(1, dtype=torch.int64, device=g.device)
        _lib.call("nvol_find_nan", _lib.ptr(g), g.numel(), _lib.ptr(first), 4, _lib.stream())
        j = int(first.item())
        return FloatingPointError(f"NaN gradient in parameter group {gi} at flat index {max(j, 0)}")

    def _nan_state(self) -> torch.Tensor:
        if getattr(self, "_nanst", None) is None:
            self._nanst = torch.tensor([NAN_NONE, 0], dtype=torch.int64, device=self.flat_params.device)
        return self._nanst

    def adam_device(self, nan_state: Optional[torch.Tensor] = None) -> None:
        """One flat Adam step (network.py:160-183) with host-cast scalars on the device
        (nvol_adam_train_step over a one-row schedule); only the parameter groups in
        front of the first one holding a NaN gradient are updated (nan_state)."""
        lr, c1, c2 = adam_scalars(self.opt, self.opt.t)
        f = lambda x: float(np.float32(x))  # noqa: E731  dt(...) of network.py:172-181
        o = self.opt
        dev = self.flat_params.device
        if getattr(self, "_adam1", None) is None:
            self._adam1 = (torch.zeros(3, dtype=torch.float32).pin_memory(), torch.zeros(3, dtype=torch.float32,
                           device=dev), torch.zeros(1, dtype=torch.int64, device=dev),
                           torch.zeros(1, dtype=torch.int32, device=dev))
        hs, sched, counter, ticket = self._adam1
        hs.numpy()[:] = (lr, c1, c2)     # train_step syncs every call: the previous copy has landed
        sched.copy_(hs, non_blocking=True)
        _lib.call("nvol_adam_train_step", _lib.ptr(self.flat_params), _lib.ptr(self.flat_grads),
                  _lib.ptr(self.flat_m), _lib.ptr(self.flat_v), self.flat_size, _lib.ptr(sched), 1,
                  _lib.ptr(counter), f(o.beta1), f(1.0 - o.beta1), f(o.beta2), f(1.0 - o.beta2), f(o.epsilon),
                  f(o.l2_reg), _lib.ptr(nan_state), None, None, 0, 0, 0.0, _lib.ptr(ticket), _lib.stream())

    def train_step(self, batch) -> float:
        """One optimization step; returns the pre-update loss (model.py:154-174).
        A NaN gradient raises FloatingPointError(group, flat index) with the groups in
        front of the offending one updated and opt.t not advanced (network.py:167-171)."""
        coords, targets = batch.coords, batch.targets
        if coords.shape[0] != self.batch_size:
            raise ConfigError(f"batch size {coords.shape[0]} != configured {self.batch_size}")
        if not self._use_kernels():
            return self._train_step_generic(coords, targets)
        c, t = self._stage_batch(coords, targets)
        if getattr(self, "_ts_bufs", None) is None:
            # the step's loss accumulator and one pinned read-back slot for [loss bits, NaN state]
            self._ts_bufs = (torch.zeros(1, dtype=torch.float64, device=c.device),
                             torch.zeros(3, dtype=torch.int64).pin_memory())
        loss_sum, back = self._ts_bufs
        loss_sum.zero_()
        ns = self._nan_state()
        self.fwd_bwd_device(c, t, loss_sum, nan_state=ns)
        self.adam_device(ns)
        back[0:1].copy_(loss_sum.view(torch.int64), non_blocking=True)   # one D2H + one sync per call
        back[1:3].copy_(ns, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        loss = float(back[0:1].view(torch.float64).item()) / c.shape[0]
        lim = int(back[1])
        if lim != NAN_NONE:
            ns.copy_(torch.tensor([NAN_NONE, 0], dtype=torch.int64))
            raise self.nan_error(lim)
        self.opt.t += 1
        return loss

    def _stage_batch(self, coords, targets):
        """Device copies of a host batch through pinned staging buffers."""
        if isinstance(coords, torch.Tensor) and coords.is_cuda:
            return coords.to(torch.float32).contiguous(), targets.to(torch.float32).contiguous()
        b = coords.shape[0]
        if self._stage is None or self._stage[0].shape[0] != b:
            dev = self.flat_params.device
            self._stage = (torch.empty((b, 3), dtype=torch.float32, device=dev),
                           torch.empty(b, dtype=torch.float32, device=dev),
                           torch.empty((b, 3), dtype=torch.float32).pin_memory(),
                           torch.empty(b, dtype=torch.float32).pin_memory())
        dc, dt_, hc, ht = self._stage
        if isinstance(coords, torch.Tensor) and coords.is_pinned() and coords.dtype == torch.float32:
            hc, ht = coords, targets                      # already pinned host tensors: DMA directly
        else:
            hc.numpy()[...] = np.asarray(coords, dtype=np.float32)
            ht.numpy()[...] = np.asarray(targets, dtype=np.float32)
        dc.copy_(hc, non_blocking=True)
        dt_.copy_(ht, non_blocking=True)
        return dc, dt_

    def _train_step_generic(self, coords, targets) -> float:
        """float64 (gradient-check) models: the modular path of model.py:159-173."""
        c, _ = to_device(coords, self.dtype)
        t, _ = to_device(targets, self.dtype)
        feats, _, _ = self.encoder.encode_device(c, check_nan=False)
        pred, acts = self.mlp.forward_device(feats)
        loss, dl = loss_and_grad(pred, t, self.loss_kind)
        dfeat = self.mlp.backward_device(acts, dl[:, None].contiguous())
        self.encoder.backward_device(c, dfeat.contiguous())
        params, grads = self.param_groups()
        adam_step(self.opt, params, grads)
        return loss

    # ---------------------------------------------------------------- inference
    def _weights_flat(self) -> torch.Tensor:
        return self.flat_params[self.w_offset:]

    def eval_device(self, coords: torch.Tensor, mode: Optional[str] = None) -> torch.Tensor:
        """Phi(coords) on the device (normalised value space)."""
        mode = mode or self.infer_mode
        if not self._use_kernels():
            feats, _, _ = self.encoder.encode_device(coords, check_nan=False)
            return self.mlp.forward_device(feats)[0]
        b = coords.shape[0]
        o = torch.empty(b, dtype=torch.float32, device=coords.device)
        if b == 0:
            return o
        c = self.encoder.config
        off, res, ent, dense = self.encoder.c_tables()
        widths = self._widths()
        relu = int(self.mlp.config.output_activation == "relu")
        if mode == "tensor":
            _lib.call("nvol_field_eval_tc", _lib.ptr(coords.contiguous()), b, _lib.ptr(self.flat_params), off, res,
                      ent, dense, c.n_levels, c.n_features_per_level, _lib.ptr(self._weights_flat()),
                      _lib.host_i32(widths), len(widths) - 1, relu, _lib.ptr(self.mlp_image()), _lib.ptr(o),
                      _lib.stream())
        else:
            _lib.call("nvol_field_eval_exact", _lib.ptr(coords.contiguous()), b, _lib.ptr(self.flat_params), off,
                      res, ent, dense, c.n_levels, c.n_features_per_level, _lib.ptr(self._weights_flat()),
                      _lib.host_i32(widths), len(widths) - 1, relu, _lib.ptr(o), _lib.stream())
        return o

    def mlp_image(self) -> torch.Tensor:
        """Device scratch the tensor-core evaluators pack the weights into (refilled on every call)."""
        if getattr(self, "_img", None) is None:
            c = self.encoder.config
            n = int(_lib.load().nvol_mlp_image_bytes(c.n_levels, c.n_features_per_level, self.mlp.config.n_neurons,
                                                      self.mlp.config.n_hidden_layers))
            if n <= 0:
                raise ConfigError("MLP shape not supported by the tcgen05 inference path")
            self._img = torch.empty(n, dtype=torch.uint8, device=self.flat_params.device)
        return self._img

    def eval_batch(self, coords):
        """Phi(coords) in normalised value space (model.py:178-182)."""
        t, host = to_device(coords, self.dtype)
        return out(self.eval_device(t), host)

    def eval_fused(self, coords):
        """Per-sample fused evaluator; bit-identical to the reference (model.py:184-198)."""
        t, host = to_device(coords, self.dtype)
        return out(self.eval_device(t, "exact"), host)

    # ---------------------------------------------------------------- config
    def config_json(self) -> dict:
        """model.py:202-214."""
        return {
            "loss": {"otype": self.loss_kind},
            "optimizer": self.opt.to_json(),
            "encoding": encoder_config_to_json(self.encoder.config),
            "network": {
                "otype": "MLP",
                "n_neurons": self.mlp.config.n_neurons,
                "n_hidden_layers": self.mlp.config.n_hidden_layers,
                "output_activation": "ReLU" if self.mlp.config.output_activation == "relu" else "None",
            },
            "batch_size": self.batch_size,
        }


def build_model(config: Optional[dict] = None, dims=(2, 2, 2), value_range=(0.0, 1.0), seed: int = 0,
                dtype=np.float32) -> NeuralModel:
    """Construct a model from a network-config dict (model.py:217-253)."""
    cfg = dict(config or {})
    loss_obj = cfg.get("loss", {"otype": "L1"})
    loss_kind = loss_obj.get("otype", "L1")
    if loss_kind not in ("L1", "L2"):
        raise ConfigError(f"unknown loss otype {loss_kind!r}; expected 'L1' or 'L2'")
    enc_cfg = encoder_config_from_json(cfg.get("encoding", {}))
    net = cfg.get("network", {})
    act = str(net.get("output_activation", "ReLU")).lower()
    if act not in ("relu", "none"):
        raise ConfigError(f"unknown output_activation {net.get('output_activation')!r}")
    rng = np.random.default_rng(seed)
    encoder = make_encoder(enc_cfg, dtype=dtype, rng=rng)
    mlp_cfg = MlpConfig(input_width=encoder.out_width, n_neurons=int(net.get("n_neurons", 64)),
                        n_hidden_layers=int(net.get("n_hidden_layers", 4)), output_activation=act)
    mlp = Mlp(mlp_cfg, dtype=dtype, rng=rng)
    opt = optimizer_from_json(cfg.get("optimizer", {}))
    return NeuralModel(encoder=encoder, mlp=mlp, opt=opt, loss_kind=loss_kind,
                       batch_size=int(cfg.get("batch_size", 65536)), value_range=tuple(value_range),
                       dims=tuple(dims))
