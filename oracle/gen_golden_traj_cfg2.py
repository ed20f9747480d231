"""Reference cfg2 loss trajectory (test infrastructure; the reference is imported read-only).

    OPENBLAS_NUM_THREADS=1 python oracle/gen_golden_traj_cfg2.py [--steps 300]

neuralvol.trainer.train(build_model(CFG2, dims=256^3, seed=0), InCoreSampler(mlobb, seed=1), steps)
(/root/reference/pkg/src/neuralvol/trainer.py:61-77) -> tests/golden/traj_cfg2.npz: the per-step
losses and learning rates, the final Adam step, per-group parameter / moment norms and a
strided sample of the final flat parameters.  Pins the device pipeline's cfg2 trajectory (the
PSNR ensemble's steps) step by step instead of only through the end-of-run PSNR.
"""
import argparse
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from neuralvol import fields  # noqa: E402
from neuralvol.model import build_model  # noqa: E402
from neuralvol.sampler import InCoreSampler  # noqa: E402
from neuralvol.trainer import train  # noqa: E402

ROOT = Path(__file__).resolve().parent.parent
CFG2 = {"encoding": {"otype": "HashGrid", "n_levels": 16, "n_features_per_level": 2,
                     "log2_hashmap_size": 19, "base_resolution": 4},
        "network": {"n_neurons": 64, "n_hidden_layers": 4}, "batch_size": 65536}
DIMS = (256, 256, 256)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--seed", type=int, default=1)
    a = ap.parse_args()
    fld = fields.rasterize("mlobb", DIMS)
    m = build_model(CFG2, dims=DIMS, seed=0)
    t0 = time.time()
    h = train(m, InCoreSampler(fld, seed=a.seed), steps=a.steps)
    print("trained", a.steps, "steps in", time.time() - t0, "s", flush=True)
    enc = np.asarray(m.encoder.params, np.float32).ravel()
    ws = [np.asarray(w, np.float32) for w in m.mlp.weights]
    flat = np.concatenate([enc] + [w.ravel() for w in ws])
    norms = [float(np.linalg.norm(enc.astype(np.float64)))] + [float(np.linalg.norm(w.astype(np.float64))) for w in ws]
    mn = [float(np.linalg.norm(np.asarray(x, np.float64))) for x in m.opt.m]
    vn = [float(np.linalg.norm(np.asarray(x, np.float64))) for x in m.opt.v]
    np.savez_compressed(ROOT / "tests" / "golden" / "traj_cfg2.npz", losses=np.asarray(h.losses),
                        lrs=np.asarray(h.lrs), steps=a.steps, seed=a.seed, t=m.opt.t, param_norms=norms,
                        m_norms=mn, v_norms=vn, flat_sample=flat[::997], n_flat=flat.size)
    print("written")


if __name__ == "__main__":
    main()
