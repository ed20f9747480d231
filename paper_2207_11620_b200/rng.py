"""Counter-based random streams for replayable rendering (the reference's rng.py API).

RngStream(seed, frame).uniform(pixel, event) draws the float32 uniforms of the path
tracer's counter stream -- a SplitMix64-style avalanche of (seed, frame, pixel, event),
24 bits, in [0, 1) -- by running the device function the tracer itself uses
(nvol_rng_u01), so host inspection and device rendering cannot drift apart.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib


@dataclass(frozen=True)
class RngStream:
    """Stateless uniform stream for one (seed, frame) pair (rng.py:43-59)."""

    seed: int
    frame: int

    def uniform(self, pixel, event):
        """float32 uniforms in [0, 1); shape follows the broadcast of pixel / event."""
        p, e = np.broadcast_arrays(np.asarray(pixel, dtype=np.uint64), np.asarray(event, dtype=np.uint64))
        shape = p.shape
        dev = _lib.device()
        tp = torch.from_numpy(np.ascontiguousarray(p.reshape(-1)).view(np.int64)).to(dev)
        te = torch.from_numpy(np.ascontiguousarray(e.reshape(-1)).view(np.int64)).to(dev)
        out = torch.empty(tp.numel(), dtype=torch.float32, device=dev)
        _lib.call("nvol_rng_u01", int(np.uint64(self.seed)), int(np.uint64(self.frame)), _lib.ptr(tp), _lib.ptr(te),
                  tp.numel(), _lib.ptr(out), _lib.stream())
        u = out.cpu().numpy().reshape(shape)
        return np.float32(u) if u.ndim == 0 else u
