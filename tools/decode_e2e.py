"""Host-landing decode (trainer.decode(..., to_host=True)) at cfg3 (1024^3): device-only decode,
the host-landing decode at several host-copy thread counts (NVOL_DECODE_HOST_THREADS), and the
raw pieces (4 GiB D2H into pinned memory; first-touch copy into a fresh numpy array)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2207_11620_b200.model import build_model  # noqa: E402
from paper_2207_11620_b200.trainer import decode  # noqa: E402

m = build_model(bench.CFG2, dims=bench.DIMS, seed=0)
m.infer_mode = os.environ.get("DECODE_MODE", "tensor")   # the bench's decode evaluator
dims = (1024, 1024, 1024)
decode(m, dims=(256, 256, 256))
torch.cuda.synchronize()
t0 = time.perf_counter()
f = decode(m, dims=dims)
torch.cuda.synchronize()
print(f"device decode {time.perf_counter() - t0:.3f} s", flush=True)
ref = float(f.data[::64, ::64, ::64].double().sum())
n = f.data.numel()
pin = torch.empty(n, dtype=torch.float32).pin_memory()
torch.cuda.synchronize()
t0 = time.perf_counter()
pin.copy_(f.data.reshape(-1), non_blocking=True)
torch.cuda.synchronize()
dt = time.perf_counter() - t0
print(f"D2H 4 GiB into pinned {dt:.3f} s ({4 * n / dt / 1e9:.1f} GB/s)", flush=True)
t0 = time.perf_counter()
o = np.empty(n, np.float32)
np.copyto(o, pin.numpy())
dt = time.perf_counter() - t0
print(f"one-thread copy into a fresh array {dt:.3f} s ({4 * n / dt / 1e9:.1f} GB/s)", flush=True)
del o, pin, f
for th in sys.argv[1:] or ["4", "8", "16"]:
    os.environ["NVOL_DECODE_HOST_THREADS"] = th
    t0 = time.perf_counter()
    h = decode(m, dims=dims, to_host=True)
    dt = time.perf_counter() - t0
    ok = abs(float(np.asarray(h.data[::64, ::64, ::64], np.float64).sum()) - ref) < 1e-6 * max(1.0, abs(ref))
    print(f"to_host threads {th}: {dt:.3f} s = {n / dt / 1e9:.2f} G samples/s, checksum {'ok' if ok else 'MISMATCH'}",
          flush=True)
    del h
