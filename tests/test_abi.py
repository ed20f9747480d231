"""CPU checks of the C-ABI boundary and host-side logic (no GPU needed)."""
from __future__ import annotations

import re
import subprocess

import numpy as np
import pytest

from conftest import ROOT


def _declared():
    text = (ROOT / "include" / "nvol.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|const char \*)\s*\**(nvol_\w+)\(", text, re.M)))


def test_library_exports_every_declared_symbol():
    from paper_2207_11620_b200 import _lib
    L = _lib.open_library()          # dlopen works without a GPU (static cudart)
    names = _declared()
    assert len(names) >= 20
    for n in names:
        assert hasattr(L, n), n
    assert set(_lib.EXPORTS) <= set(names) | {"nvol_last_error"}
    assert L.nvol_abi_version() == 4


def test_library_is_sm100a():
    so = ROOT / "paper_2207_11620_b200" / "lib" / "libnvol.so"
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(so)], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2207_11620_b200 import _lib
    with pytest.raises(RuntimeError, match="CUDA"):
        _lib.load()


def test_pcg64_state_and_shard_offsets():
    # host side of the device sampler: initial state words and DP row offsets
    from paper_2207_11620_b200.sampler import PcgStream
    s = PcgStream(1)
    assert hex(s.state) == "0x9c5b484bfedb756c2a6e7d6f320fbc7e"
    assert hex(s.inc) == "0x922af2da2645f895a19857b95740937b"
    # the u32 offset of rank r's shard of step k equals the rows it would see
    # in the single-process batch (verified numerically by the oracle stream)
    import nvol_oracle as orc
    B, G, k = 64, 4, 3
    full = orc.pcg64_random_f32(1, 3 * B * k, 3 * B).reshape(B, 3)
    for r in range(G):
        part = orc.pcg64_random_f32(1, 3 * B * k + 3 * (B // G) * r, 3 * (B // G)).reshape(B // G, 3)
        np.testing.assert_array_equal(part, full[r * (B // G):(r + 1) * (B // G)])


def test_config_validation_mirrors_reference():
    from paper_2207_11620_b200.encoding import EncoderConfig, level_resolution
    from paper_2207_11620_b200.errors import ConfigError
    from paper_2207_11620_b200.network import MlpConfig, OptimizerState, lr_at
    with pytest.raises(ConfigError):
        EncoderConfig(kind="hashgrid", n_features_per_level=3)
    with pytest.raises(ConfigError):
        EncoderConfig(kind="hashgrid", log2_hashmap_size=9)
    with pytest.raises(ConfigError):
        EncoderConfig(kind="nope")
    with pytest.raises(ConfigError):
        MlpConfig(input_width=8, n_neurons=24)
    assert level_resolution(EncoderConfig(n_levels=4), 3) == 32
    assert EncoderConfig(kind="frequency").out_width == 192
    opt = OptimizerState()
    assert lr_at(opt, 3000) == pytest.approx(0.005 * 0.99)


def test_hash_index_known_answers():
    from paper_2207_11620_b200.encoding import hash_index
    assert hash_index(125, 4, (1, 2, 3)) == 86
    assert hash_index(125, 4, (0, 0, 0)) == 0
    assert hash_index(125, 4, (4, 4, 4)) == 124
    # u32 wrap before the modulo (test_encoding.py:107-111)
    v = (4000, 3999, 4001)
    h = 0
    for a, p in enumerate((1, 2654435761, 805459861)):
        h ^= (v[a] * p) & 0xFFFFFFFF
    assert hash_index(1021, 4096, v, dense=False) == h % 1021


def test_vnr_header_roundtrip_host(tmp_path):
    # byte layout of the model file without touching the device
    import json
    import struct
    from paper_2207_11620_b200.trainer import MODEL_MAGIC, MODEL_VERSION
    cfg = {"a": 1, "n_params": 3}
    payload = json.dumps(cfg, sort_keys=True).encode()
    raw = MODEL_MAGIC + struct.pack("<II", MODEL_VERSION, len(payload)) + payload + np.ones(3, "<f4").tobytes()
    assert raw[:4] == b"VNRM" and struct.unpack("<II", raw[4:12]) == (1, len(payload))


def test_binding_arity_matches_header():
    """Every ctypes signature in _lib has exactly the parameter count the header
    declares (a missing argument would be passed with ctypes' default int
    conversion -- a truncated pointer on the device path)."""
    from paper_2207_11620_b200 import _lib
    text = (ROOT / "include" / "nvol.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    decls = {m.group(1): m.group(2) for m in re.finditer(r"\b(nvol_\w+)\s*\(([^;{]*?)\)\s*;", text, re.S)}
    for name, args in _lib._SIGS.items():
        assert name in decls, name
        params = decls[name].strip()
        n = 0 if params in ("", "void") else params.count(",") + 1
        assert n == len(args), (name, n, len(args))
