"""Out-of-core sampler golden vectors from the REAL reference (build container only).

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python oracle/gen_golden_outofcore.py

sampler.py:86-297 BlockBuffer / sample_outofcore on the reference's own test
volume recipe (test_sampler.py disk_volume: default_rng(5).random((16,20,32))
as float32, value_range (0,1)): R=8, S=3, block 8^3, buffer rng default_rng(5),
sampling rng default_rng(6), four batches of 1024 with a refresh after each
(test_sampler.py:297-308).  Writes tests/golden/outofcore.npz.
"""
from __future__ import annotations

import sys
import tempfile
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from neuralvol.sampler import BlockBuffer, sample_outofcore  # noqa: E402
from neuralvol.volume import ScalarField, VolumeMeta, save_volume  # noqa: E402

OUT = Path(__file__).resolve().parent.parent / "tests" / "golden" / "outofcore.npz"


def main():
    dims = (32, 20, 16)
    data = np.random.default_rng(5).random((16, 20, 32)).astype(np.float32)
    f = ScalarField(VolumeMeta(dims=dims, dtype="f32", value_range=(0.0, 1.0)), data)
    with tempfile.TemporaryDirectory() as d:
        side = Path(d) / "vol.json"
        save_volume(f, side)
        buf = BlockBuffer(side, r=8, s=3, rng=np.random.default_rng(5), block_dims=(8, 8, 8))
        rng = np.random.default_rng(6)
        cs, ts, origins = [], [], []
        for _ in range(4):
            b = sample_outofcore(buf, 1024, rng)
            cs.append(b.coords)
            ts.append(b.targets)
            origins.append(buf.origins.copy())
            buf.refresh()
        buf.join()
        np.savez_compressed(OUT, coords=np.stack(cs), targets=np.stack(ts), origins=np.stack(origins),
                            final_origins=buf.origins, generations=buf.generations, payloads=buf.payloads)
        buf.close()
    print(OUT)


if __name__ == "__main__":
    main()
