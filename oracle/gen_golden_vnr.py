"""Golden .vnr written by the reference -- test infrastructure (SURVEY.md §8 f4 wire formats).

    python oracle/gen_golden_vnr.py      # -> tests/golden/ref_cfg1.vnr + tests/golden/vnr_cfg1.npz

The reference (/root/reference/pkg/src/neuralvol, imported read-only) trains its cfg1
model 200 steps on mlobb 48^3 with a non-unit value range, writes it with
trainer.save_model (trainer.py:125-138), and records eval_fused on fixed coordinates
and decode() on a small grid, so the GPU tests can load the reference's file, check
the evaluations, and check that save_model here writes the same bytes back.
"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from neuralvol import fields  # noqa: E402
from neuralvol.model import build_model  # noqa: E402
from neuralvol.sampler import InCoreSampler  # noqa: E402
from neuralvol.trainer import decode, save_model, train  # noqa: E402

OUT = Path(__file__).resolve().parent.parent / "tests" / "golden"
CFG1 = {"encoding": {"otype": "HashGrid", "n_levels": 4, "n_features_per_level": 2,
                     "log2_hashmap_size": 12, "base_resolution": 4},
        "network": {"n_neurons": 16, "n_hidden_layers": 2}, "batch_size": 8192}

f = fields.rasterize("mlobb", (48, 48, 48))
m = build_model(CFG1, dims=(48, 48, 48), value_range=(2.0, 5.0), seed=0)
train(m, InCoreSampler(f, seed=1), steps=200)
save_model(m, OUT / "ref_cfg1.vnr")
coords = np.random.default_rng(8).random((2048, 3)).astype(np.float32)
dec = decode(m, dims=(20, 16, 12))
np.savez_compressed(OUT / "vnr_cfg1.npz", coords=coords, eval_fused=m.eval_fused(coords),
                    eval_batch=m.eval_batch(coords), decode=dec.data, dims=np.array([20, 16, 12]))
print("wrote", OUT / "ref_cfg1.vnr", (OUT / "ref_cfg1.vnr").stat().st_size, "bytes")
