"""Diagnostics: tcgen05 vs fp32 SIMT vs oracle gradients (per level / per layer)."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))
sys.path.insert(0, str(ROOT / "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import nvol_oracle as orc  # noqa: E402
from conftest import golden, golden_config  # noqa: E402
from paper_2207_11620_b200.model import build_model  # noqa: E402


def rel_l2(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


for name in ("cfg1", "cfg2"):
    for loss in ("L2", "L1"):
        cfg = dict(golden_config(golden(f"encode_{name}.npz")), batch_size=8192, loss={"otype": loss})
        ref = orc.OracleModel(cfg, seed=0)
        norm = orc.rasterize("mlobb", (32, 32, 32))
        c, t = orc.InCoreSampler(norm, seed=1).sample(8192)
        cap = {}
        want = ref.train_step(c, t, capture=cap)
        res, ent, dense, off = orc.level_tables(ref.spec)
        for mode in (0, 1):
            m = build_model(cfg, dims=(32, 32, 32), seed=0)
            m.train_mode = mode
            acc = torch.zeros(1, dtype=torch.float64, device="cuda")
            m.fwd_bwd_device(torch.from_numpy(c).cuda(), torch.from_numpy(t).cuda(), acc)
            g = m.encoder.param_grads.cpu().numpy()
            per = [rel_l2(g[off[l]:off[l] + ent[l] * 2], cap["enc_grads"][off[l]:off[l] + ent[l] * 2])
                   for l in range(len(res))]
            mlp = [rel_l2(x.cpu().numpy(), y) for x, y in zip(m.mlp.grads, cap["w_grads"])]
            print(f"{name} {loss} mode{mode} loss {float(acc.item())/8192:.6f} ref {want:.6f} "
                  f"enc {rel_l2(g, cap['enc_grads']):.4f} per-level {np.round(per, 4).tolist()} "
                  f"mlp {np.round(mlp, 4).tolist()}", flush=True)
