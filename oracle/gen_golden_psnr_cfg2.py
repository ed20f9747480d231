"""Reference PSNR ensembles (cfg2 = the bench's training config; cfg1 = the survey's
capacity-limited protocol) -- test infrastructure.

    OPENBLAS_NUM_THREADS=1 python oracle/gen_golden_psnr_cfg2.py [--cfg cfg1] --seed S [--steps N]   # one member
    python oracle/gen_golden_psnr_cfg2.py [--cfg cfg1] --merge      # -> tests/golden/psnr_<cfg>_mlobb.json
    python oracle/gen_golden_psnr_cfg2.py --append                 # add the PART members to the fixture

SURVEY.md §8(c) protocol at configs[1]: the reference's cfg2 model (HashGrid 16 x 2^19 x 2,
4 x 64 ReLU MLP, B = 65,536, L1 + Adam; model seed 0) trained with
`neuralvol.trainer.train(model, InCoreSampler(field, seed=S), steps)` on
`fields.rasterize("mlobb", (256,)*3)` for sampler seeds 1..5, then
`psnr(field, decode(model))` at 256^3 (/root/reference/pkg/src/neuralvol/trainer.py:61-106,
volume.py:197-242).  Reduced step count (the reference runs at ~0.8 s per cfg2 step on
one core); the number of steps and the BLAS thread count are recorded in the fixture.
Each member runs in its own process (the members are independent) so the ensemble
finishes in one member's time on a multi-core host.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

OUT = Path(__file__).resolve().parent.parent / "tests" / "golden"
PART = Path(os.environ.get("PSNR_PARTS", "/tmp/psnr_cfg2_parts"))
CFG2 = {"encoding": {"otype": "HashGrid", "n_levels": 16, "n_features_per_level": 2,
                     "log2_hashmap_size": 19, "base_resolution": 4},
        "network": {"n_neurons": 64, "n_hidden_layers": 4}, "batch_size": 65536}
DIMS = (256, 256, 256)
CFG1 = {"encoding": {"otype": "HashGrid", "n_levels": 4, "n_features_per_level": 2,
                     "log2_hashmap_size": 12, "base_resolution": 4},
        "network": {"n_neurons": 16, "n_hidden_layers": 2}, "batch_size": 65536}
SETUPS = {"cfg2": (CFG2, DIMS), "cfg1": (CFG1, (64, 64, 64))}


def member(seed: int, steps: int, cfg_name: str = "cfg2") -> None:
    cfg, dims = SETUPS[cfg_name]
    sys.path.insert(0, "/root/reference/pkg/src")
    from neuralvol import fields
    from neuralvol.model import build_model
    from neuralvol.sampler import InCoreSampler
    from neuralvol.trainer import decode, train
    from neuralvol.volume import psnr
    fld = fields.rasterize("mlobb", dims)
    model = build_model(cfg, dims=dims, seed=0)
    t0 = time.time()
    hist = train(model, InCoreSampler(fld, seed=seed), steps=steps)
    t1 = time.time()
    val = float(psnr(fld, decode(model, dims=dims)))
    PART.mkdir(exist_ok=True)
    (PART / f"{cfg_name}_seed{seed}.json").write_text(json.dumps(
        {"seed": seed, "steps": steps, "psnr": val, "final_loss": float(hist.losses[-1]),
         "losses": [float(x) for x in hist.losses],
         "train_s": t1 - t0, "decode_s": time.time() - t1,
         "openblas_num_threads": os.environ.get("OPENBLAS_NUM_THREADS", "unset")}))
    print("seed", seed, "psnr", val, flush=True)


def merge(cfg_name: str = "cfg2") -> None:
    cfg, dims = SETUPS[cfg_name]
    parts = sorted((json.loads(p.read_text()) for p in PART.glob(f"{cfg_name}_seed*.json")), key=lambda d: d["seed"])
    vals = [p["psnr"] for p in parts]
    steps = {p["steps"] for p in parts}
    threads = {p["openblas_num_threads"] for p in parts}
    assert len(steps) == 1 and len(threads) == 1, (steps, threads)
    name = os.environ.get("PSNR_OUT", f"psnr_{cfg_name}_mlobb.json")
    (OUT / name).write_text(json.dumps(
        {"config": cfg, "field": "mlobb", "dims": list(dims), "steps": steps.pop(), "model_seed": 0,
         "sampler_seeds": [p["seed"] for p in parts], "psnr_db": vals, "mean": float(np.mean(vals)),
         "std": float(np.std(vals)), "final_losses": [p["final_loss"] for p in parts],
         "openblas_num_threads": threads.pop(), "reference_train_s": [p["train_s"] for p in parts],
         "generator": "oracle/gen_golden_psnr_cfg2.py (neuralvol.trainer.train + decode + volume.psnr)"}, indent=1))


def append(cfg_name: str = "cfg2") -> None:
    """Extend an existing fixture with the members in PART (same steps / BLAS threads), keeping
    their per-step loss trajectories as 500-step block means (loss_block_means)."""
    path = OUT / os.environ.get("PSNR_OUT", f"psnr_{cfg_name}_mlobb.json")
    g = json.loads(path.read_text())
    parts = sorted((json.loads(p.read_text()) for p in PART.glob(f"{cfg_name}_seed*.json")), key=lambda d: d["seed"])
    for p in parts:
        assert p["steps"] == g["steps"] and p["openblas_num_threads"] == g["openblas_num_threads"], p["seed"]
        assert p["seed"] not in g["sampler_seeds"], p["seed"]
        g["sampler_seeds"].append(p["seed"])
        g["psnr_db"].append(p["psnr"])
        g["final_losses"].append(p["final_loss"])
        g["reference_train_s"].append(p["train_s"])
        g.setdefault("loss_block_means", {})[str(p["seed"])] = [
            float(x) for x in np.asarray(p["losses"]).reshape(-1, 500).mean(1)]
    g["loss_block"] = 500
    g["mean"], g["std"] = float(np.mean(g["psnr_db"])), float(np.std(g["psnr_db"]))
    path.write_text(json.dumps(g, indent=1))


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--seed", type=int)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--merge", action="store_true")
    ap.add_argument("--append", action="store_true")
    ap.add_argument("--cfg", default="cfg2", choices=sorted(SETUPS))
    a = ap.parse_args()
    if a.merge:
        merge(a.cfg)
    elif a.append:
        append(a.cfg)
    else:
        member(a.seed, a.steps, a.cfg)
