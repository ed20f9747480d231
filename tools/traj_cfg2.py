"""cfg2 loss trajectory per training engine against the reference's (tests/golden/traj_cfg2.npz,
oracle/gen_golden_traj_cfg2.py) -- diagnostic.

    python tools/traj_cfg2.py [--steps 300]
"""
import argparse
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

CFG2 = {"encoding": {"otype": "HashGrid", "n_levels": 16, "n_features_per_level": 2, "log2_hashmap_size": 19,
                     "base_resolution": 4}, "network": {"n_neurons": 64, "n_hidden_layers": 4}, "batch_size": 65536}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--modes", default="0,1")
    a = ap.parse_args()
    from paper_2207_11620_b200 import fields, trainer
    from paper_2207_11620_b200.model import build_model
    from paper_2207_11620_b200.sampler import InCoreSampler
    z = np.load(ROOT / "tests" / "golden" / "traj_cfg2.npz")
    ref = z["losses"]
    n = min(a.steps, ref.size)
    dims = (256,) * 3
    fld = fields.rasterize("mlobb", dims, host=True)
    for mode in [int(x) for x in a.modes.split(",")]:
        m = build_model(CFG2, dims=dims, seed=0)
        m.train_mode = mode
        h = trainer.train(m, InCoreSampler(fld, seed=int(z["seed"])), steps=n)
        got = np.asarray(h.losses)
        enc = m.encoder.params.detach().double().cpu().numpy().ravel()
        ws = [w.detach().double().cpu().numpy() for w in m.mlp.weights]
        flat = np.concatenate([enc.astype(np.float32)] + [w.astype(np.float32).ravel() for w in ws])
        norms = [float(np.linalg.norm(enc))] + [float(np.linalg.norm(w)) for w in ws]
        mn = [float(np.linalg.norm(x.detach().double().cpu().numpy())) for x in m.opt.m]
        vn = [float(np.linalg.norm(x.detach().double().cpu().numpy())) for x in m.opt.v]
        pick = [0, 1, 2, 3, 5, 10, 20, 30, 50, 75, 100, 150, 200, 250, n - 1]
        rows = {k: [float(got[k]), float(ref[k]), float(got[k] / ref[k] - 1)] for k in pick if k < n}
        w = 25
        sm = lambda x: np.convolve(x, np.ones(w) / w, mode="valid")
        print(json.dumps({"mode": mode, "per_step": rows,
                          "smoothed_rel": [float(x) for x in (sm(got[:n]) / sm(ref[:n]) - 1)[::w]],
                          "param_norms": [norms, [float(x) for x in z["param_norms"]]],
                          "m_norms": [mn, [float(x) for x in z["m_norms"]]],
                          "v_norms": [vn, [float(x) for x in z["v_norms"]]],
                          "flat_sample_rel_l2": float(np.linalg.norm(flat[::997] - z["flat_sample"]) /
                                                      np.linalg.norm(z["flat_sample"])),
                          "t": [int(m.opt.t), int(z["t"])]}), flush=True)


if __name__ == "__main__":
    main()
