"""Benchmark: cfg2 hash-grid + MLP training step (BASELINE.json configs[1]).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Own arm: K device-resident training steps (sample -> fused fwd/bwd ->
[NCCL all-reduce] -> flat Adam, one CUDA graph per step) of the cfg2 model
(16 levels x 2^19 x 2 features, 4x64 ReLU MLP, B = 65,536 samples/step, L1 +
Adam) on a synthetic 256^3 mlobb volume, timed with CUDA events, max over
ranks.  Data parallel runs shard the fixed global batch (strong scaling,
bit-identical sample stream to the single-GPU run).  Prints ONE JSON line.

Reference arm: the CPU oracle (the reference's algorithm restated in C +
numpy/OpenBLAS, oracle/) on all host cores, same config / metric.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CFG2 = {"loss": {"otype": "L1"},
        "encoding": {"otype": "HashGrid", "n_levels": 16, "n_features_per_level": 2,
                     "log2_hashmap_size": 19, "base_resolution": 4, "per_level_scale": 2.0},
        "network": {"otype": "MLP", "n_neurons": 64, "n_hidden_layers": 4, "output_activation": "ReLU"},
        "batch_size": 65536}
DIMS = (256, 256, 256)
FIELD = "mlobb"
METRIC = "train samples/s (hash-grid+fused-MLP step)"
PEAKS_PATH = ROOT / "MEASURED_PEAKS.json"


def peaks():
    try:
        p = json.loads(PEAKS_PATH.read_text())
        return p["hbm_gbs"], p["bf16_tflops_sustained"], p.get("bf16_tflops", 1644.6), "measured"
    except Exception:
        return 6650.0, 1400.0, 1590.0, "fallback"


# ---------------------------------------------------------------------------- clocks

class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.lines = []
        if self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()
                out = ""
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in getattr(self, "lines", []):
            f = [x.strip() for x in l.split(",")]
            try:
                sm.append(float(f[0]))
                mx = max(mx, float(f[1]))
                for n, v in zip(names, f[2:]):
                    if v.lower() == "active":
                        reasons.add(n)
            except (ValueError, IndexError):
                continue
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------- CPU oracle

def cpu_train_rate(steps: int, budget_s: float = 30.0):
    """Oracle (reference algorithm on host cores) cfg2 training throughput."""
    sys.path.insert(0, str(ROOT / "oracle"))
    import nvol_oracle as orc
    orc.build()
    norm = orc.rasterize(FIELD, DIMS)
    model = orc.OracleModel(CFG2, seed=0)
    sampler = orc.InCoreSampler(norm, seed=1)
    B = model.batch_size
    c, t = sampler.sample(B)
    t0 = time.perf_counter()
    model.train_step(c, t)                      # warm-up (BLAS / page faults)
    one = time.perf_counter() - t0
    n = max(1, min(steps, int(budget_s / max(one, 1e-3))))
    t0 = time.perf_counter()
    for _ in range(n):
        c, t = sampler.sample(B)
        model.train_step(c, t)
    dt = time.perf_counter() - t0
    threads = max(orc.num_threads(), int(os.environ.get("OPENBLAS_NUM_THREADS", os.cpu_count() or 1)))
    return {"value": B * n / dt, "unit": "samples/s", "cores": int(threads), "kind": "port",
            "sample": f"{n} full cfg2 training steps (B=65536, sampling + encode + MLP + loss + scatter + dense Adam "
                      f"over 12,181,394 params) of the C/numpy oracle, {dt:.2f} s"}


# ---------------------------------------------------------------------------- reference arm

def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    r = cpu_train_rate(args.steps, budget_s=120.0)
    line = {"impl": "reference", "metric": METRIC, "value": r["value"], "unit": "samples/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 65536 / r["value"] * 1e3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": "cfg2 training step: 256^3 mlobb, HashGrid 16x2^19x2, 4x64 MLP, B=65536, L1+Adam"},
            "cpu_baseline": r,
            "e2e": {"value": r["value"], "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------- own arm

def run_ours(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2207_11620_b200 import _lib, fields
    from paper_2207_11620_b200.model import build_model
    from paper_2207_11620_b200.sampler import InCoreSampler, SampleBatch
    from paper_2207_11620_b200.trainer import StepPipeline, decode

    L = _lib.load()
    hbm, tc_sus, tc_burst, peak_kind = peaks()
    mode = args.mode
    model = build_model(CFG2, dims=DIMS, seed=0)
    model.train_mode = mode
    field = fields.rasterize(FIELD, DIMS)
    sampler = InCoreSampler(field, seed=1)
    B = model.batch_size
    K, W = args.steps, args.warmup
    pipe = StepPipeline(model, sampler, capacity=K + W + 2, rank=rank, world=world)
    stream = torch.cuda.current_stream()

    # ---- warm-up (includes graph capture)
    pipe.step(W)
    torch.cuda.synchronize()

    # ---- timed region: K graph replays
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(stream)
        pipe.step(K)
        ev1.record(stream)
        torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.barrier()
    losses = pipe.finish()
    ms_per_step = ms / K
    value = B * K / (ms / 1e3)

    # ---- per-phase device times (instrumented eager steps, same kernels as the graph)
    phases = {"sample": [], "fwd_bwd": [], "adam": []}
    vol = sampler.volume
    dz, dy, dx = vol.shape
    for _ in range(5):
        e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        e[0].record(stream)
        _lib.call("nvol_sample_incore_dev", *sampler.rng.words(), pipe.u32_base, _lib.ptr(pipe.counter), pipe.t0, B,
                  pipe.row0, pipe.b, _lib.ptr(vol), dx, dy, dz, _lib.ptr(pipe.coords), _lib.ptr(pipe.targets),
                  _lib.stream())
        e[1].record(stream)
        model.fwd_bwd_device(pipe.coords, pipe.targets, pipe.acc, b_global=B)
        e[2].record(stream)
        _lib.call("nvol_adam_flat_dev", _lib.ptr(model.flat_params), _lib.ptr(model.flat_grads), _lib.ptr(model.flat_m),
                  _lib.ptr(model.flat_v), model.flat_size, _lib.ptr(pipe.sched), pipe.sched.numel() // 3,
                  _lib.ptr(pipe.counter), *pipe.adam_consts, _lib.ptr(pipe.nan_flag), _lib.stream())
        e[3].record(stream)
        torch.cuda.synchronize()
        phases["sample"].append(e[0].elapsed_time(e[1]))
        phases["fwd_bwd"].append(e[1].elapsed_time(e[2]))
        phases["adam"].append(e[2].elapsed_time(e[3]))
    ph = {k: float(np.median(v)) for k, v in phases.items()}
    n_flat = model.flat_size
    adam_bytes = 32 * n_flat
    m_lv, nf = 16, 2
    gather_bytes = B * m_lv * 8 * nf * 4
    scatter_bytes = 2 * gather_bytes
    mlp_flops = 3 * 2 * B * (32 * 64 + 3 * 64 * 64 + 64)
    dominant = max(ph, key=ph.get)
    if dominant == "adam":
        ach = adam_bytes / (ph["adam"] * 1e-3) / 1e9
        roof = {"kernel": "adam_flat_kernel", "bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s",
                "frac": ach / hbm, "traffic": None, "algorithmic_bytes_per_launch": adam_bytes,
                "peak_source": peak_kind}
    elif dominant == "fwd_bwd":
        byts = gather_bytes + scatter_bytes + B * 16
        ach = byts / (ph["fwd_bwd"] * 1e-3) / 1e9
        roof = {"kernel": "train_fwd_bwd (encode gather + MLP + scatter)", "bound": "hbm", "achieved": ach,
                "peak": hbm, "unit": "GB/s", "frac": ach / hbm, "traffic": None,
                "algorithmic_bytes_per_launch": byts, "peak_source": peak_kind,
                "mlp_tflops": mlp_flops / (ph["fwd_bwd"] * 1e-3) / 1e12}
    else:
        byts = B * 48
        ach = byts / (ph["sample"] * 1e-3) / 1e9
        roof = {"kernel": "sample_incore_kernel", "bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s",
                "frac": ach / hbm, "traffic": None, "algorithmic_bytes_per_launch": byts, "peak_source": peak_kind}
    step_bytes = adam_bytes + gather_bytes + scatter_bytes + B * 64
    roof["step_algorithmic_bytes"] = step_bytes
    roof["step_frac_of_hbm"] = step_bytes / (ms_per_step * 1e-3) / 1e9 / hbm

    # ---- e2e through the public API with host (pinned) buffers
    e2e = None
    if world == 1:
        e2e_steps = max(3, min(K, 50))
        host = []
        for _ in range(e2e_steps + 2):
            bt = sampler.sample(B)
            host.append((bt.coords.cpu().pin_memory(), bt.targets.cpu().pin_memory()))
        model.train_step(SampleBatch(*host[0], trusted=True))
        model.train_step(SampleBatch(*host[1], trusted=True))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for k in range(e2e_steps):
            model.train_step(SampleBatch(*host[k + 2], trusted=True))
        dt = time.perf_counter() - t0
        e2e = {"value": B * e2e_steps / dt, "unit": "samples/s", "h2d_bytes_per_step": B * 3 * 4 + B * 4,
               "d2h_bytes_per_step": 8, "api": "NeuralModel.train_step(SampleBatch(host pinned coords, targets))",
               "steps": e2e_steps}

    # ---- decode (cfg3 shape, reported beside the headline)
    dec = None
    if world == 1 and not args.no_decode:
        dd = (args.decode_dim,) * 3
        model.infer_mode = args.decode_mode
        decode(model, dims=(64, 64, 64))
        torch.cuda.synchronize()
        d0, d1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        d0.record(stream)
        out = decode(model, dims=dd)
        d1.record(stream)
        torch.cuda.synchronize()
        dms = d0.elapsed_time(d1)
        nvox = dd[0] * dd[1] * dd[2]
        dec = {"value": nvox / (dms / 1e3), "unit": "samples/s", "ms": dms, "dims": list(dd),
               "mode": args.decode_mode, "mlp_tflops": nvox * 2 * (32 * 64 + 3 * 64 * 64 + 64) / (dms * 1e-3) / 1e12}
        del out

    launches = pipe.launches_per_step() * K
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_train_rate(3, budget_s=args.cpu_budget)

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": world, "steps": K, "warmup": W,
                "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                "config": {"workload": "cfg2 training step (configs[1]): synthetic 256^3 mlobb volume, HashGrid "
                                       "16 levels x 2^19 x 2 feat, 4x64 ReLU MLP, B=65536/step global, L1 + Adam",
                           "global_batch": B, "parallelism": f"dp{world}", "mode": "tcgen05" if mode else "simt",
                           "l2": "inputs larger than L2: each step streams 390 MB of Adam state (> 126 MB L2)"},
                "phases_ms": ph, "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
                "clocks": clk.summary(), "decode": dec, "final_loss": float(losses[-1])}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--mode", type=int, default=int(os.environ.get("NVOL_TRAIN_MODE", "0")))
    ap.add_argument("--decode-dim", type=int, default=512)
    ap.add_argument("--decode-mode", default="exact")
    ap.add_argument("--no-decode", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
