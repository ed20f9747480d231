"""Online macro-cell golden vectors from the REAL reference (build container only).

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python oracle/gen_golden_online.py

macrocell.py:101-133 macrocell_update_online applied to five InCoreSampler
batches (seed 3) of a 24x20x16 blobs field with 4-voxel cells: writes the
batches and the resulting value_lo / value_hi to tests/golden/macrocell_online.npz.
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from neuralvol import fields  # noqa: E402
from neuralvol.macrocell import macrocell_empty, macrocell_update_online  # noqa: E402
from neuralvol.sampler import InCoreSampler  # noqa: E402

OUT = Path(__file__).resolve().parent.parent / "tests" / "golden" / "macrocell_online.npz"


def main():
    dims = (24, 20, 16)
    fld = fields.rasterize("blobs", dims)
    grid = macrocell_empty(dims, n_g=4)
    s = InCoreSampler(fld, seed=3)
    cs, ts = [], []
    for _ in range(5):
        b = s.sample(4096)
        macrocell_update_online(grid, b)
        cs.append(b.coords)
        ts.append(b.targets)
    np.savez_compressed(OUT, coords=np.stack(cs), targets=np.stack(ts), lo=grid.value_lo, hi=grid.value_hi,
                        dims=np.array(dims), n_g=4)
    print(OUT, grid.value_lo.shape)


if __name__ == "__main__":
    main()
