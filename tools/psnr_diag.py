"""cfg2 ensemble diagnostic: per engine and sampler seed, the end-of-run PSNR, the final loss and
loss statistics over the run (the reference's fixture records PSNR and final loss per seed).

    python tools/psnr_diag.py --seeds 16 --modes 0,1
"""
import argparse
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seeds", type=int, default=16)
    ap.add_argument("--steps", type=int, default=3000)
    ap.add_argument("--modes", default="0,1")
    a = ap.parse_args()
    from paper_2207_11620_b200 import fields, trainer
    from paper_2207_11620_b200.model import build_model
    from paper_2207_11620_b200.sampler import InCoreSampler
    from paper_2207_11620_b200.volume import psnr
    g = json.loads((ROOT / "tests" / "golden" / "psnr_cfg2_mlobb.json").read_text())
    dims = tuple(g["dims"])
    fld = fields.rasterize(g["field"], dims, host=True)
    for mode in [int(x) for x in a.modes.split(",")]:
        rows = []
        for seed in range(1, a.seeds + 1):
            m = build_model(g["config"], dims=dims, seed=0)
            m.train_mode = mode
            h = trainer.train(m, InCoreSampler(fld, seed=seed), steps=a.steps)
            l = np.asarray(h.losses)
            rows.append({"seed": seed, "psnr": float(psnr(fld, trainer.decode(m, dims=dims))),
                         "final": float(l[-1]), "mean_last500": float(l[-500:].mean()),
                         "med_last500": float(np.median(l[-500:])), "max_last500": float(l[-500:].max()),
                         "mean_by_500": [float(x) for x in l.reshape(-1, 500).mean(1)]})
        ps = np.array([r["psnr"] for r in rows])
        print(json.dumps({"mode": mode, "psnr_mean": float(ps.mean()), "psnr_std": float(ps.std(ddof=1)),
                          "final_mean": float(np.mean([r["final"] for r in rows])),
                          "mean_last500": float(np.mean([r["mean_last500"] for r in rows])),
                          "rows": rows}), flush=True)
    print(json.dumps({"reference": {"psnr": g["psnr_db"], "final": g["final_losses"]}}))


if __name__ == "__main__":
    main()
