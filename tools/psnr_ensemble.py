"""cfg1 PSNR ensemble (SURVEY §8c protocol): mlobb 64^3, 2000 steps, model seed 0, sampler
seeds 1-5, per engine; compare with the reference's ensemble (tests/golden/psnr_cfg1_mlobb.json)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2207_11620_b200 import fields, trainer
from paper_2207_11620_b200.model import MODE_TCGEN05, build_model
from paper_2207_11620_b200.sampler import InCoreSampler
from paper_2207_11620_b200.volume import psnr
g = json.load(open(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "psnr_cfg1_mlobb.json")))
dims = tuple(g["dims"])
fld = fields.rasterize(g["field"], dims, host=True)
for mode in (0, MODE_TCGEN05):
    res = []
    t0 = time.time()
    for seed in g["sampler_seeds"]:
        m = build_model(g["config"], dims=dims, seed=g["model_seed"])
        m.train_mode = mode
        trainer.train(m, InCoreSampler(fld, seed=seed), steps=g["steps"])
        res.append(psnr(fld, trainer.decode(m, dims=dims)))
    print(json.dumps({"mode": mode, "psnr": res, "mean": float(np.mean(res)), "ref_mean": g["mean"],
                      "delta": float(np.mean(res) - g["mean"]), "s": time.time() - t0}))
