"""Benchmark: cfg2 hash-grid + MLP training step (BASELINE.json configs[1]).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Own arm: K device-resident training steps (sample -> encode / tcgen05 MLP /
scatter (three streams) -> [NCCL all-reduce] -> flat Adam; one CUDA graph per
step) of the cfg2 model (16 levels x 2^19 x 2 features, 4x64 ReLU MLP,
B = 65,536 samples/step, L1 + Adam) on a synthetic 256^3 mlobb volume, timed
with CUDA events, max over ranks.  Data-parallel runs shard the fixed global
batch (strong scaling; the union of the shards is the single-process batch).
Prints ONE JSON line; decode (cfg3) and render (cfg4) rates ride along in
sub-objects.

Reference arm: the CPU oracle (the reference's algorithm restated in C +
numpy/OpenBLAS, oracle/) on all host threads, same config / metric.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import subprocess
import sys
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
N_PARAMS_CFG2 = 12_181_394


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
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            time.sleep(0.3)  # let the sampler start before the timed region
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
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
        for l in self.lines:
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
            "sample": f"{n} full cfg2 training steps (B=65536: sampling + encode + MLP + loss + scatter + dense Adam "
                      f"over 12,181,394 params) of the C/numpy oracle in {dt:.2f} s on {threads} threads"}


def cpu_decode_rate(model_blob, n: int = 48):
    """Oracle eval_batch (the reference decode path) on an n^3 brick of the cfg2 model."""
    sys.path.insert(0, str(ROOT / "oracle"))
    import nvol_oracle as orc
    m = orc.OracleModel(CFG2, seed=0)
    m.load_flat(model_blob)
    t0 = time.perf_counter()
    orc.decode(m, (n, n, n), slab_z=8)
    dt = time.perf_counter() - t0
    return {"value": n ** 3 / dt, "unit": "samples/s", "sample": f"{n}^3 voxel decode (eval_batch path)",
            "cores": orc.num_threads(), "kind": "port"}


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

def _event_ms(torch, fn, reps=5, nev=2):
    """Device time of fn() with CUDA events on the current stream; a spin
    kernel in front keeps the host ahead of the GPU so launch latency is
    excluded."""
    out = []
    for _ in range(reps):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(nev)]
        for e in ev:          # torch creates the CUDA event lazily on first record
            e.record()
        torch.cuda.synchronize()
        torch.cuda._sleep(2_000_000)
        fn(ev)
        torch.cuda.synchronize()
        out.append([ev[0].elapsed_time(e) for e in ev[1:]])
    return np.median(np.array(out), axis=0)


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2207_11620_b200 import _lib, fields
    from paper_2207_11620_b200.distributed import init_from_env
    from paper_2207_11620_b200.model import build_model
    from paper_2207_11620_b200.sampler import InCoreSampler, SampleBatch
    from paper_2207_11620_b200.trainer import StepPipeline, decode

    rank, world, local = init_from_env("nccl")
    if world != args.gpus:
        raise SystemExit(f"bench.py --gpus {args.gpus} but the process group has {world} rank(s)")
    torch.cuda.set_device(local)
    _lib.load()
    comm = {"backend": dist.get_backend() if world > 1 else None, "world": world,
            "nccl_version": ".".join(map(str, torch.cuda.nccl.version())) if world > 1 else None}
    hbm, tc_sus, tc_burst, peak_kind = peaks()
    model = build_model(CFG2, dims=DIMS, seed=0)
    model.train_mode = args.mode
    field = fields.rasterize(FIELD, DIMS)
    sampler = InCoreSampler(field, seed=1)
    B = model.batch_size
    K, W = args.steps, args.warmup
    pipe = StepPipeline(model, sampler, capacity=K + W + 2, rank=rank, world=world)
    stream = torch.cuda.current_stream()

    pipe.step(W)                      # warm-up (the second step captures the graph)
    torch.cuda.synchronize()
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

    # ---- per-kernel device times: CUDA events on the launching stream
    vol = sampler.volume
    dz, dy, dx = vol.shape
    b = pipe.b

    def sample_fn(ev):
        ev[0].record(stream)
        _lib.call("nvol_sample_incore_dev", *sampler.rng.words(), pipe.u32_base, _lib.ptr(pipe.counter), pipe.t0, B,
                  pipe.row0, b, _lib.ptr(vol), dx, dy, dz, _lib.ptr(pipe.coords), _lib.ptr(pipe.targets),
                  _lib.stream())
        ev[1].record(stream)

    def stages_fn(ev):
        arr = (__import__("ctypes").c_void_p * 4)(*[e.cuda_event for e in ev[:4]])
        _lib.call("nvol_set_stage_events", arr, 4)
        model.fwd_bwd_device(pipe.coords, pipe.targets, pipe.acc, b_global=B)
        ev[4].record(stream)
        _lib.call("nvol_set_stage_events", None, 0)

    def adam_fn(ev):
        ev[0].record(stream)
        _lib.call("nvol_adam_train_step", _lib.ptr(model.flat_params), _lib.ptr(model.flat_grads),
                  _lib.ptr(model.flat_m), _lib.ptr(model.flat_v), model.flat_size, _lib.ptr(pipe.sched),
                  pipe.sched.numel() // 3, _lib.ptr(pipe.counter), *pipe.adam_consts, _lib.ptr(pipe.nan_state),
                  _lib.ptr(pipe.acc), None, pipe.t0, 0, 1.0 / B, _lib.ptr(pipe.ticket), _lib.stream())
        ev[1].record(stream)

    def fused_fn(ev):
        cfg = model.encoder.config
        off, res, ent, dense = model.encoder.c_tables()
        ws = model._workspace(b)
        ev[0].record(stream)
        _lib.call("nvol_adam_encode_step", _lib.ptr(model.flat_params), _lib.ptr(model.flat_grads),
                  _lib.ptr(model.flat_m), _lib.ptr(model.flat_v), model.flat_size, _lib.ptr(pipe.sched),
                  pipe.sched.numel() // 3, _lib.ptr(pipe.counter), *pipe.adam_consts, _lib.ptr(pipe.nan_state),
                  _lib.ptr(pipe.acc), None, pipe.t0, 0, 1.0 / B, _lib.ptr(pipe.work), _lib.ptr(pipe.bufs[1][0]), b,
                  off, res, ent, dense, cfg.n_levels, cfg.n_features_per_level, model.mlp.config.n_neurons,
                  model.mlp.config.n_hidden_layers, _lib.ptr(ws), ws.numel(), _lib.stream())
        ev[1].record(stream)

    def exchange_fn(ev):
        from paper_2207_11620_b200.distributed import allgather_shards, reduce_scatter_grads
        ev[0].record(stream)
        if pipe.sharded:
            reduce_scatter_grads(model.flat_grads_padded, pipe.gslice, None)
            allgather_shards(model.flat_params_padded, rank, None)
        else:
            dist.all_reduce(model.flat_grads)
        ev[1].record(stream)

    exchange = None
    if world > 1 and getattr(pipe, "peer", None) is not None:
        exchange = {"kind": "peer-memory fused reduce-scatter + Adam + all-gather (csrc/dp_peer.cu, NVOL_DP_PEER=1)",
                    "ms": None, "note": "inside the step (one kernel per rank); ms_per_step includes it"}
    elif world > 1:
        snap = model.flat_params.clone()
        t_x = float(_event_ms(torch, exchange_fn)[0])
        model.flat_params.copy_(snap)
        model.flat_grads.zero_()
        t = torch.tensor([t_x], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        exchange = {"ms": float(t.item()), "bytes_per_rank": 4 * model.flat_size * (2 if pipe.sharded else 1),
                    "kind": "NCCL reduce-scatter + all-gather (sharded optimizer)" if pipe.sharded
                    else "NCCL all-reduce", "share_of_step": float(t.item()) / ms_per_step}
    # the kernels the step launches (nvol_train_fwd_bwd / nvol_adam_train_step pick them; the
    # NVOL_MLP4 / NVOL_ADAM_TMA switches select the previous designs for A/B runs)
    K_ADAM = "adam_step_kernel" if os.environ.get("NVOL_ADAM_TMA", "1") == "0" else "adam_tma_kernel"
    K_MLP = "mlp_tc_kernel" if os.environ.get("NVOL_MLP4", "1") == "0" else "mlp_tc4_kernel"
    t_sample = float(_event_ms(torch, sample_fn)[0])
    t_adam = float(_event_ms(torch, adam_fn)[0])
    kernels = {"sample_incore_kernel": t_sample, K_ADAM: t_adam}
    if pipe.fused:
        kernels["adam_encode_kernel"] = float(_event_ms(torch, fused_fn)[0])
    if args.mode == 1:
        st = _event_ms(torch, stages_fn, nev=5)
        kernels.update({"encode_tiles_kernel": float(st[0]), K_MLP: float(st[1] - st[0]),
                        "scatter_kernel": float(st[2] - st[1])})
    n_flat = model.flat_size
    adam_bytes = 32 * n_flat
    gather_bytes = B * 16 * 8 * 2 * 4
    mlp_flops = 3 * 2 * B * (32 * 64 + 3 * 64 * 64 + 64)
    # roofline of the dominant single kernel
    dom = max(kernels, key=kernels.get)
    per_unit = {K_ADAM: (adam_bytes, "hbm", "32 B/param x 12,181,396 flat params"),
                "scatter_kernel": (2 * gather_bytes, "hbm", "16 levels x 8 corners x 2 feat x 4 B x 2 (RMW) per sample"),
                "encode_tiles_kernel": (gather_bytes + B * 12 + B * 64 * 2, "hbm",
                                        "1,024 B gathered + 12 B coords + 128 B fp16 tiles per sample"),
                "sample_incore_kernel": (B * 48, "hbm", "48 B per sample"),
                "adam_encode_kernel": (adam_bytes + gather_bytes + B * 12 + B * 64 * 2, "hbm",
                                       "32 B/param Adam x 12,181,396 flat params + the next batch's encode "
                                       "(1,024 B gathered + 12 B coords + 128 B fp16 tiles per sample)")}
    if dom in per_unit:
        byts, bound, how = per_unit[dom]
        ach = byts / (kernels[dom] * 1e-3) / 1e9
        roof = {"kernel": dom, "bound": bound, "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm,
                "traffic": None, "algorithmic_bytes_per_launch": byts, "algorithmic_basis": how,
                "launch_ms": kernels[dom], "peak_source": peak_kind}
    else:
        ach = mlp_flops / (kernels[dom] * 1e-3) / 1e12
        roof = {"kernel": dom, "bound": "tensor", "achieved": ach, "peak": tc_sus, "unit": "TFLOP/s",
                "frac": ach / tc_sus, "traffic": None, "algorithmic_flops_per_launch": mlp_flops,
                "launch_ms": kernels[dom], "peak_source": peak_kind}
    # DRAM traffic of the dominant kernel per launch, from the committed ncu --set full capture
    # (profiles/ncu_traffic.json, written from profiles/<round>_ncu_summary.md)
    try:
        tr = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "ncu_traffic.json")))
        if dom in tr:
            roof["traffic"] = tr[dom]["traffic_bytes"]
            roof["traffic_source"] = tr["_source"]
    except (OSError, ValueError, KeyError):
        pass
    step_bytes = adam_bytes + 3 * gather_bytes + B * 64
    roof["step_algorithmic_bytes"] = step_bytes
    roof["step_frac_of_hbm"] = step_bytes / (ms_per_step * 1e-3) / 1e9 / hbm
    roof["kernel_ms"] = kernels
    if args.mode == 1:
        roof["mlp_tc_tflops"] = mlp_flops / (kernels[K_MLP] * 1e-3) / 1e12
    # every step kernel against the peak that bounds it; the L2 denominators are
    # measured live (nvol_l2_probe: random 8-byte gathers / float2 REDs into a
    # 48 MB L2-resident region), the HBM and tensor ones are MEASURED_PEAKS.json
    probe = (ctypes.c_double * 3)()
    _lib.call("nvol_l2_probe", probe)
    l2_stream, l2_gather, l2_red = float(probe[0]), float(probe[1]), float(probe[2])
    m_lv, n_coarse = 16, 3          # cfg2: levels 0-2 (46 KB) accumulate in shared memory in the scatter
    rl = {"l2_peaks_measured": {"stream_read_gbs": l2_stream, "gather8_gops": l2_gather, "red_gops": l2_red}}
    if args.mode == 1:
        enc_ops = B * m_lv * 8
        rl["encode_tiles_kernel"] = {"bound": "l2 gather rate", "achieved_gops": enc_ops / (kernels["encode_tiles_kernel"] * 1e-3) / 1e9,
                                     "peak_gops": l2_gather, "basis": "B x 16 levels x 8 corner gathers"}
        rl["encode_tiles_kernel"]["frac"] = rl["encode_tiles_kernel"]["achieved_gops"] / l2_gather
        sc_ops = B * (m_lv - n_coarse) * 8
        rl["scatter_kernel"] = {"bound": "l2 RED rate", "achieved_gops": sc_ops / (kernels["scatter_kernel"] * 1e-3) / 1e9,
                                "peak_gops": l2_red, "basis": "B x 13 global levels x 8 corner updates"}
        rl["scatter_kernel"]["frac"] = rl["scatter_kernel"]["achieved_gops"] / l2_red
        rl[K_MLP] = {"bound": "tensor", "achieved_tflops": roof["mlp_tc_tflops"], "peak_tflops": tc_sus,
                               "frac": roof["mlp_tc_tflops"] / tc_sus,
                               "note": "M=128 x N=64 tcgen05 MMAs issue at <= 2725 MAC/clk/SM (67% of the 4096 peak, "
                                       "tools/micro/mma_bench.cu); the chain of 8 dependent layer phases per tile is "
                                       "latency-bound"}
    rl[K_ADAM] = {"bound": "hbm", "achieved_gbs": adam_bytes / (kernels[K_ADAM] * 1e-3) / 1e9, "peak_gbs": hbm}
    rl[K_ADAM]["frac"] = rl[K_ADAM]["achieved_gbs"] / hbm
    if "adam_encode_kernel" in kernels:
        t_ae = kernels["adam_encode_kernel"]
        rl["adam_encode_kernel"] = {"bound": "hbm (Adam stream) + l2 gathers (encode), overlapped",
                                    "achieved_adam_gbs": adam_bytes / (t_ae * 1e-3) / 1e9, "peak_gbs": hbm,
                                    "frac": adam_bytes / (t_ae * 1e-3) / 1e9 / hbm,
                                    "vs_separate_ms": t_adam + kernels.get("encode_tiles_kernel", 0.0),
                                    "basis": "Adam bytes only: the encode runs in the shadow of the Adam sweep"}
    roof["rooflines"] = rl

    # ---- e2e through the public API with host (pinned) buffers: trainer.train()
    # over a sampler that hands out host batches; every step DMAs its 1 MB batch
    # from pinned memory and reads its loss back (async, pinned), wall clock
    e2e = None
    if world == 1:
        from paper_2207_11620_b200.trainer import train
        e2e_steps = max(200, min(K, 500))   # amortises the per-call sync of train() like a real run
        host = []
        for _ in range(e2e_steps + 4):
            bt = sampler.sample(B)
            host.append(SampleBatch(bt.coords.cpu().pin_memory(), bt.targets.cpu().pin_memory(), trusted=True))

        class _HostBatches:
            """sampler.py:263-297 protocol over pre-made pinned host batches."""
            def __init__(self, batches):
                self.batches, self.i = batches, 0

            def sample(self, b):
                bt = self.batches[self.i % len(self.batches)]
                self.i += 1
                return bt

        hs = _HostBatches(host)
        train(model, hs, steps=4)                 # warm-up: builds the pipeline, captures its two graphs
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        hist = train(model, hs, steps=e2e_steps)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        e2e = {"value": B * e2e_steps / dt, "unit": "samples/s", "h2d_bytes_per_step": B * 3 * 4 + B * 4,
               "d2h_bytes_per_step": 8, "steps": e2e_steps, "ms_per_step": dt * 1e3 / e2e_steps,
               "api": "trainer.train(model, sampler over pinned host batches, steps): per step H2D of coords+targets "
                      "(copy stream, overlapped with the previous step) and D2H of the step loss",
               "final_loss": float(hist.losses[-1])}
        # the reference's per-call API as well: NeuralModel.train_step(batch) -> float (a sync per step)
        model.train_step(host[0])
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for k in range(20):
            model.train_step(host[1 + k])
        dt = time.perf_counter() - t0
        e2e["train_step_api"] = {"value": B * 20 / dt, "unit": "samples/s", "steps": 20}

    # ---- the fp32 SIMT engine (ordered-reduction / bitwise-repeatable mode's engine) on the same step
    simt = None
    if args.mode == 1 and world == 1 and not args.no_simt:
        ms_s = simt_rate(torch, model, sampler, K=min(K, 20))
        simt = {"value": B / (ms_s * 1e-3), "unit": "samples/s", "ms_per_step": ms_s,
                "engine": "fp32 SIMT (generic kernels, CUDA cores; what set_deterministic(True) runs)"}

    # ---- decode (cfg3) and render (cfg4) beside the headline
    dec = None
    if not args.no_decode:
        # cfg3: z-slab bricks sharded over the ranks (distributed.decode_shard), no exchange;
        # device time per rank with CUDA events, max over ranks
        from paper_2207_11620_b200.distributed import decode_shard
        dd = (args.decode_dim,) * 3
        model.infer_mode = args.decode_mode
        decode(model, dims=(64, 64, 64))
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        d0, d1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        d0.record(stream)
        z0, out = decode_shard(model, dd, rank, world)
        d1.record(stream)
        torch.cuda.synchronize()
        dms = d0.elapsed_time(d1)
        if world > 1:
            t = torch.tensor([dms], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dms = float(t.item())
        nvox = dd[0] * dd[1] * dd[2]
        live = decode_live_corners(model, dd)
        vps = nvox / (dms / 1e3)
        flops_vox = 2 * (32 * 64 + 3 * 64 * 64 + 64)
        dec = {"value": vps, "unit": "samples/s", "ms": dms, "dims": list(dd),
               "mode": args.decode_mode, "workload": "cfg3: full-grid decode of the cfg2 model",
               "sharding": f"z-slabs over {world} GPU(s), max over ranks",
               "roofline": {"bound": "l2 gather rate (encoder) / tensor (MLP)",
                            "live_corner_gathers_per_voxel": live,
                            "achieved_gather_gops": live * vps / 1e9, "peak_gather_gops": l2_gather,
                            "frac": live * vps / 1e9 / l2_gather,
                            "mlp_tflops": vps * flops_vox / 1e12, "mlp_peak_tflops": tc_sus,
                            "mlp_frac": vps * flops_vox / 1e12 / tc_sus,
                            "hbm_bytes_per_voxel": 4, "hbm_frac": vps * 4 / 1e9 / hbm,
                            "basis": "corners with non-zero trilinear weight at voxel centres (zero-weight corners "
                                     "are skipped bit-exactly); 28,800 algorithmic MLP flop per voxel"}}
        del out
        if world == 1:
            # e2e through the public API: decode(model, dims, to_host=True) lands the 4 GiB volume in
            # host memory (per-slab D2H overlapped with the next slab's decode, host copies over
            # worker threads), as the reference's decode returns a host ScalarField
            # (trainer.py:98-106); wall clock of the second call (the first one allocates the pinned
            # staging slabs, which torch's host allocator then caches), incl. the output array
            del decode(model, dims=dd, to_host=True).data
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            fld_h = decode(model, dims=dd, to_host=True)
            wall = time.perf_counter() - t0
            dec["e2e"] = {"value": nvox / wall, "unit": "samples/s", "s": wall, "h2d_bytes": 0,
                          "d2h_bytes": nvox * 4, "api": "trainer.decode(model, dims, to_host=True) -> host "
                                                        "ScalarField (numpy f32)", "call": "second (warm pinned staging)",
                          "checksum": float(np.asarray(fld_h.data[::64, ::64, ::64], np.float64).sum())}
            del fld_h
        if rank == 0 and world == 1 and not args.no_cpu:
            dec["cpu_baseline"] = cpu_decode_rate(model.blob().cpu().numpy())
    rend = None
    if not args.no_render:
        rend = render_bench(torch, args, rank, world)
        wt = rend.get("wavefront_tensor") if rend else None
        if wt:
            # the frame against the L2 random-gather ceiling of its field evaluations: every
            # evaluation at an arbitrary position gathers 16 levels x 8 corners (whole frame,
            # marching and compaction included; the evaluator kernel alone is in DESIGN.md)
            g = wt["evals_per_s"] * 16 * 8 / 1e9
            rend["roofline"] = {"bound": "l2 gather rate (field evaluations)", "gathers_per_eval": 128,
                                "achieved_gather_gops": g, "peak_gather_gops": l2_gather, "frac": g / l2_gather,
                                "basis": "wavefront_tensor frame: evaluations/s x 128 corner gathers, whole frame"}
    c5 = None
    if not args.no_cfg5:
        c5 = cfg5_bench(torch, args, rank, world)

    launches = pipe.launches_per_step() * K
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_train_rate(3, budget_s=args.cpu_budget)

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": world, "steps": K, "warmup": W,
                "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None,
                "dtype": ("f32 tables / loss / Adam; fp16-operand tcgen05 MLP (split-fp16 forward, fp16 backward, "
                          "fp32 accumulate)") if args.mode == 1 else "f32",
                "data": "synthetic",
                "config": {"workload": "cfg2 training step (configs[1]): synthetic 256^3 mlobb volume, HashGrid "
                                       "16 levels x 2^19 x 2 feat, 4x64 ReLU MLP, B=65536/step global, L1 + Adam",
                           "global_batch": B, "parallelism": f"dp{world}",
                           "engine": "tcgen05 (split-fp16 forward, fp16 backward, fp32 accumulate)" if args.mode
                           else "simt fp32",
                           "l2": "inputs larger than L2: each step streams 390 MB of Adam state (> 126 MB L2)"},
                "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
                "clocks": clk.summary(), "decode": dec, "render": rend, "cfg5": c5, "simt_engine": simt,
                "exchange": exchange, "comm": comm,
                "final_loss": float(losses[-1])}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def decode_live_corners(model, dims) -> float:
    """Mean number of corners with non-zero trilinear weight per voxel-centre sample
    ((i+0.5)/D per axis) over the levels -- the gathers the decode actually issues."""
    res = [int(r) for r in model.encoder.level_resolutions]
    tot = 0.0
    for r in res:
        per_axis = []
        for d in dims:
            i = np.arange(d, dtype=np.float32)
            p = (i + np.float32(0.5)) / np.float32(d)
            s = p * np.float32(r)
            fr = s - np.floor(s)
            per_axis.append(float(np.mean(np.where(fr == 0, 1.0, 2.0))))
        tot += per_axis[0] * per_axis[1] * per_axis[2]
    return tot


def simt_rate(torch, model0, sampler, K=20):
    """ms per device-resident cfg2 step of the fp32 SIMT engine (same model shape / batch)."""
    from paper_2207_11620_b200.model import MODE_SIMT, build_model
    from paper_2207_11620_b200.trainer import StepPipeline
    m = build_model(CFG2, dims=DIMS, seed=0)
    m.train_mode = MODE_SIMT
    p = StepPipeline(m, sampler, capacity=K + 4)
    p.step(3)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s = torch.cuda.current_stream()
    e0.record(s)
    p.step(K)
    e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / K
    p.finish()
    del p, m
    return ms


def cfg5_bench(torch, args, rank=0, world=1):
    """configs[4]: the 2048x2048x1920 (RM-T60-sized) synthetic volume, rasterised on the
    device (f32, 30 GiB, HBM-resident on every rank), trained with the cfg2 network by
    the same data-parallel pipeline (rank r samples rows [r*B/G, (r+1)*B/G)); the
    global batch stays 65,536.  Device-timed K steps, max over ranks."""
    import torch.distributed as dist
    from paper_2207_11620_b200 import fields
    from paper_2207_11620_b200.model import build_model
    from paper_2207_11620_b200.sampler import InCoreSampler
    from paper_2207_11620_b200.trainer import StepPipeline
    dims = (2048, 2048, 1920)
    t0 = time.perf_counter()
    fld = fields.rasterize(FIELD, dims)
    vol = fld.normalized
    torch.cuda.synchronize()
    rast_s = time.perf_counter() - t0
    m = build_model(CFG2, dims=dims, seed=0)
    m.train_mode = args.mode
    K = max(10, min(args.steps, 50))
    pipe = StepPipeline(m, InCoreSampler(fld, seed=1), capacity=K + 4, rank=rank, world=world)
    pipe.step(3)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s = torch.cuda.current_stream()
    e0.record(s)
    pipe.step(K)
    e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    losses = pipe.finish()
    res = {"workload": "cfg5: 2048x2048x1920 mlobb volume (f32, device-rasterised, 30 GiB per GPU), cfg2 network, "
                       f"B=65536 global, data-parallel over {world} GPU(s)",
           "value": m.batch_size * K / (ms * 1e-3), "unit": "samples/s", "ms_per_step": ms / K, "steps": K,
           "rasterize_s": rast_s, "volume_gib": vol.numel() * 4 / 2 ** 30, "final_loss": float(losses[-1])}
    del pipe, m, fld, vol
    torch.cuda.empty_cache()
    return res


def render_bench(torch, args, rank=0, world=1):
    """cfg4: 1920x1080 macro-cell ray march of a cfg2 model trained on blobs 256^3
    (image row tiles over the ranks, distributed.render_tile; max over ranks)."""
    from paper_2207_11620_b200 import fields
    from paper_2207_11620_b200.camera import default_camera
    from paper_2207_11620_b200.macrocell import macrocell_from_model, macrocell_set_tf
    from paper_2207_11620_b200.model import build_model
    from paper_2207_11620_b200.render import RenderConfig
    from paper_2207_11620_b200.sampler import InCoreSampler
    from paper_2207_11620_b200.trainer import train
    from paper_2207_11620_b200.transfer import default_tf
    fld = fields.rasterize("blobs", DIMS)
    m = build_model(CFG2, dims=DIMS, seed=0)
    m.train_mode = args.mode
    train(m, InCoreSampler(fld, seed=1), steps=args.render_train_steps)
    tf = default_tf()
    macrocell_from_model(m, n_g=16)          # warm-up (module load, scratch)
    torch.cuda.synchronize()
    g0 = time.perf_counter()
    grid = macrocell_from_model(m, n_g=16)
    macrocell_set_tf(grid, tf)
    torch.cuda.synchronize()
    mc_ms = (time.perf_counter() - g0) * 1e3
    cam = default_camera(DIMS, 1920, 1080)
    cfg = RenderConfig(mode="raymarch", use_macrocells=True, k_batch=8, step_size=1.0, max_step=64.0)
    res = {"workload": "cfg4: 1920x1080 raymarch, macro-cells n_g=16, K=8, step 1, cfg2 model trained "
                       f"{args.render_train_steps} steps on blobs 256^3, default TF/camera",
           "macrocell_from_model_ms": mc_ms}
    from paper_2207_11620_b200.distributed import render_tile
    import torch.distributed as dist
    res["sharding"] = f"image row tiles over {world} GPU(s), frame time = max over ranks"
    for arch, mode in (("wavefront", "tensor"), ("reference", "tensor"), ("wavefront", "exact"), ("reference", "exact")):
        render_tile(m, tf, cam, cfg, grid, rank, world, arch, mode)       # warm-up
        torch.cuda.synchronize()
        ts = []
        for _ in range(3):
            if world > 1:
                dist.barrier()
            t0 = time.perf_counter()
            _, img, st = render_tile(m, tf, cam, cfg, grid, rank, world, arch, mode)
            torch.cuda.synchronize()
            ts.append((time.perf_counter() - t0) * 1e3)
        fms, evals = float(np.median(ts)), st.evals
        if world > 1:
            t = torch.tensor([fms, float(evals)], dtype=torch.float64, device="cuda")
            dist.all_reduce(t[:1], op=dist.ReduceOp.MAX)
            e = t[1:].clone()
            dist.all_reduce(e, op=dist.ReduceOp.SUM)
            fms, evals = float(t[0].item()), int(e.item())
        res[f"{'inshader' if arch == 'reference' else arch}_{mode}"] = {"frame_ms": fms, "fps": 1e3 / fms, "evals": evals,
                                 "evals_per_s": evals / (fms * 1e-3), "iterations": len(st.alive_per_iteration)}
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--mode", type=int, default=int(os.environ.get("NVOL_TRAIN_MODE", "1")))
    ap.add_argument("--decode-dim", type=int, default=1024)
    ap.add_argument("--decode-mode", default="tensor")
    ap.add_argument("--render-train-steps", type=int, default=300)
    ap.add_argument("--no-decode", action="store_true")
    ap.add_argument("--no-render", action="store_true")
    ap.add_argument("--no-cfg5", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-simt", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: relaunch under the torchrun launcher (rendezvous on 127.0.0.1)
        import socket
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), str(Path(__file__).resolve())] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
