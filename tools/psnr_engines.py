"""PSNR ensembles per training engine (diagnostic): SIMT fp32, tcgen05 two-slot (NVOL_MLP4=0 in a
child process) and tcgen05 four-slot, on a given config / field / steps.

    python tools/psnr_engines.py --cfg cfg2 --dims 48 --batch 16384 --steps 200 --seeds 8
"""
import argparse
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

CFGS = {
    "cfg1": {"encoding": {"otype": "HashGrid", "n_levels": 4, "n_features_per_level": 2, "log2_hashmap_size": 12,
                          "base_resolution": 4}, "network": {"n_neurons": 16, "n_hidden_layers": 2}},
    "cfg2": {"encoding": {"otype": "HashGrid", "n_levels": 16, "n_features_per_level": 2, "log2_hashmap_size": 19,
                          "base_resolution": 4}, "network": {"n_neurons": 64, "n_hidden_layers": 4}},
}


def run(a, mode):
    import numpy as np
    from paper_2207_11620_b200 import fields, trainer
    from paper_2207_11620_b200.model import build_model
    from paper_2207_11620_b200.sampler import InCoreSampler
    from paper_2207_11620_b200.volume import psnr
    dims = (a.dims,) * 3
    cfg = dict(CFGS[a.cfg], batch_size=a.batch)
    fld = fields.rasterize(a.field, dims, host=True)
    res = []
    for seed in range(1, a.seeds + 1):
        m = build_model(cfg, dims=dims, seed=0)
        m.train_mode = mode
        trainer.train(m, InCoreSampler(fld, seed=seed), steps=a.steps)
        res.append(psnr(fld, trainer.decode(m, dims=dims)))
    return {"mode": mode, "mlp4": os.environ.get("NVOL_MLP4", "1"), "mean": float(np.mean(res)),
            "std": float(np.std(res, ddof=1)), "psnr": res}


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", default="cfg2")
    ap.add_argument("--dims", type=int, default=48)
    ap.add_argument("--field", default="mlobb")
    ap.add_argument("--batch", type=int, default=16384)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--seeds", type=int, default=8)
    ap.add_argument("--child", type=int, default=-1)
    a = ap.parse_args()
    if a.child >= 0:
        print(json.dumps(run(a, a.child)))
        sys.exit(0)
    base = [sys.executable, __file__] + [x for x in sys.argv[1:]]
    for mode, env in ((0, "1"), (1, "0"), (1, "1")):
        out = subprocess.run(base + ["--child", str(mode)], env=dict(os.environ, NVOL_MLP4=env), capture_output=True,
                             text=True)
        print(out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-500:], flush=True)
