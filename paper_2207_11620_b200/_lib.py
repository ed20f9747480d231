"""ctypes binding of libnvol.so (the C ABI declared in include/nvol.h).

There is no CPU fallback: every compute entry point of the package goes
through this module, and loading fails loudly when the library or a CUDA
device is missing.
"""
from __future__ import annotations

import ctypes
from pathlib import Path

import numpy as np
import torch

from .errors import ConfigError

LIB_PATH = Path(__file__).resolve().parent / "lib" / "libnvol.so"
_lib = None

P = ctypes.c_void_p
I32, I64, U64, F32, F64 = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_float, ctypes.c_double

# name -> argtypes (restype int unless listed in _RESTYPES)
_SIGS = {
    "nvol_abi_version": [],
    "nvol_last_error": [],
    "nvol_has_tcgen05": [I32],
    "nvol_set_deterministic": [I32],
    "nvol_grid_encode_fwd": [P, I64, P, P, P, P, P, I32, I32, P, P, P, I32, P],
    "nvol_grid_encode_bwd": [P, P, P, I64, I32, I32, P, I32, P],
    "nvol_grid_encode_bwd_coords": [P, P, I64, P, P, P, P, I32, I32, P, I32, I32, P],
    "nvol_mlp_forward": [I64, I32, P, P, P, I32, I32, P],
    "nvol_mlp_backward": [I64, I32, P, P, P, P, P, P, P, P, I32, I32, P],
    "nvol_loss_and_grad": [P, P, I64, I32, P, P, I32, P],
    "nvol_loss_and_grad_scaled": [P, P, I64, I64, I32, P, P, I32, P],
    "nvol_loss_record": [P, P, P, I64, I64, F64, P],
    "nvol_adam_step": [P, P, P, P, I64] + [F64] * 9 + [I32, P],
    "nvol_find_nan": [P, I64, P, I32, P],
    "nvol_sample_incore": [U64, U64, U64, U64, U64, I64, P, I64, I64, I64, P, P, P],
    "nvol_sample_incore_dev": [U64, U64, U64, U64, U64, P, I64, I64, I64, I64, P, I64, I64, I64, P, P, P],
    "nvol_sample_incore_dev_mc": [U64, U64, U64, U64, U64, P, I64, I64, I64, I64, P, I64, I64, I64, P, P, P, P,
                                  I64, I64, I64, I64, P],
    "nvol_macrocell_update_online": [P, P, I64, I64, I64, I64, P, P, I64, I64, I64, I64, P],
    "nvol_sample_outofcore": [P, P, P, I64, P, P, P, I64, I64, I64, I64, I64, I64, I32, P, P, P],
    "nvol_trilinear": [P, I64, I64, I64, P, I64, P, P],
    "nvol_rasterize": [I32, I64, I64, I64, I64, I64, P, I32, P],
    "nvol_sq_err_sum": [P, P, I64, P, P],
    "nvol_field_eval_exact": [P, I64, P, P, P, P, P, I32, I32, P, P, I32, I32, P, P],
    "nvol_field_eval_tc": [P, I64, P, P, P, P, P, I32, I32, P, P, I32, I32, P, P, P],
    "nvol_mlp_image_bytes": [I32, I32, I32, I32],
    "nvol_decode": [P, P, P, P, P, I32, I32, P, P, I32, I32, I64, I64, I64, I64, I64, F64, F64, P, I32, P, P],
    "nvol_train_fwd_bwd": [P, P, I64, I64, P, P, P, P, P, P, I32, I32, I32, I32, I32, I32, P, P, I64, I32, P, P],
    "nvol_nan_scan": [P, I64, P, I32, P, P],
    "nvol_train_workspace_bytes": [I64, I32, I32, I32, I32, I32],
    "nvol_train_tc_supported": [I32, I32, I32, I32],
    "nvol_adam_flat_dev": [P, P, P, P, I64, P, I64, P, F32, F32, F32, F32, F32, F32, P, P],
    "nvol_adam_train_step": [P, P, P, P, I64, P, I64, P, F32, F32, F32, F32, F32, F32, P, P, P, I64, I64, F64, P,
                             P],
    "nvol_adam_encode_step": [P, P, P, P, I64, P, I64, P, F32, F32, F32, F32, F32, F32, P, P, P, I64, I64, F64, P,
                              P, I64, P, P, P, P, I32, I32, I32, I32, P, I64, P],
    "nvol_render_workspace_bytes": [I64, I32],
    "nvol_set_stage_events": [P, I32],
    "nvol_set_fork_event": [P],
    "nvol_dp_signal": [P, P, P, P],
    "nvol_dp_wait": [I32, P, P, P, P, P],
    "nvol_dp_fused_adam": [I32, I32, P, P, P, P, P, I64, I64, P, P, P, I64, P, F32, F32, F32, F32, F32, F32, P, P,
                           I64, I64, F64, P, P],
    "nvol_train_tc_debug": [P, P, P],
    "nvol_train_tc_scatter": [P, P, I64, I64, P, P, P, P, I32, I32, P, P],
    "nvol_l2_persist": [I64],
    "nvol_l2_probe": [P],
    "nvol_render": [P, P, P, P, I32, P, P, I32, P, I64, I64, I64, I32, P, I64, I64, I64, P, P, P, P, P, I32, I32,
                    P, P, I32, I32, I32, I32, P, P, P, I64, P, P, I32, P],
    "nvol_macrocell_ranges": [P, I64, I64, I64, I64, I32, P, P, P],
    "nvol_macrocell_set_tf": [P, P, I64, P, P, I32, F64, P, P],
    "nvol_rng_u01": [U64, U64, P, P, I64, P, P],
    "nvol_march_formula": [I32, P, I64, F32, F32, F32, P, P],
    "nvol_dda_collect": [P, F64, F64, F64, I64, I64, I64, I64, P, P, P, P],
}
_RESTYPES = {"nvol_last_error": ctypes.c_char_p, "nvol_train_workspace_bytes": I64, "nvol_mlp_image_bytes": I64,
             "nvol_l2_persist": I64,
             "nvol_render_workspace_bytes": I64}

EXPORTS = tuple(_SIGS)


def open_library(path: Path | str = LIB_PATH):
    """dlopen libnvol.so and attach signatures (works without a GPU)."""
    if not Path(path).exists():
        raise RuntimeError(f"libnvol.so not built at {path}; run __graft_entry__.build()")
    L = ctypes.CDLL(str(path))
    for name, args in _SIGS.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = _RESTYPES.get(name, ctypes.c_int)
    return L


def load():
    """The library, with a CUDA device present; raises otherwise (no CPU fallback)."""
    global _lib
    if _lib is None:
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2207_11620_b200 needs a CUDA (sm_100a) device; none is visible")
        _lib = open_library()
    return _lib


def check(status: int, what: str = "") -> None:
    if status == 0:
        return
    msg = (load().nvol_last_error() or b"").decode()
    if status == 1:
        raise ConfigError(f"{what}: {msg}" if what else msg)
    raise RuntimeError(f"{what}: CUDA error: {msg}" if what else msg)


def call(name: str, *args) -> None:
    fn = getattr(load(), name)
    if len(args) != len(fn.argtypes):   # ctypes would pass extras with int conversion (truncated pointers)
        raise TypeError(f"{name}: {len(args)} arguments for {len(fn.argtypes)} parameters")
    check(fn(*args), name)


def ptr(t) -> int | None:
    if t is None:
        return None
    return t.data_ptr()


def stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def host_i64(a) -> ctypes.Array:
    a = np.ascontiguousarray(a, dtype=np.int64)
    return (ctypes.c_int64 * len(a))(*a.tolist())


def host_u8(a) -> ctypes.Array:
    a = np.ascontiguousarray(a, dtype=np.uint8)
    return (ctypes.c_uint8 * len(a))(*a.tolist())


def host_i32(a) -> ctypes.Array:
    a = list(int(x) for x in a)
    return (ctypes.c_int32 * len(a))(*a)


def host_ptrs(ts) -> ctypes.Array:
    return (ctypes.c_void_p * len(ts))(*[t.data_ptr() for t in ts])


def dtype_bytes(dtype) -> int:
    if dtype in (torch.float32, np.float32) or dtype == np.dtype(np.float32):
        return 4
    if dtype in (torch.float64, np.float64) or dtype == np.dtype(np.float64):
        return 8
    raise ConfigError(f"unsupported dtype {dtype}; expected float32 or float64")


def device() -> torch.device:
    return torch.device("cuda", torch.cuda.current_device())
