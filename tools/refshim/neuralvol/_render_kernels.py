"""The reference's render-kernel module surface the reference tests touch: _u01, the path
tracer's counter uniform (_render_kernels.py:42-49), served by the device function the
tracer uses (paper_2207_11620_b200.rng / nvol_rng_u01)."""
import numpy as np

from paper_2207_11620_b200.rng import RngStream


def _u01(seed, frame, pixel, event):
    return np.float32(RngStream(int(seed), int(frame)).uniform(np.uint64(pixel), np.uint64(event)))
