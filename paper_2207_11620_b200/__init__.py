"""paper_2207_11620_b200: B200-native instant neural volume representation.

From-scratch sm_100a implementation of the hash-grid encoder + ReLU MLP
training step, full-grid decode and macro-cell ray marching of arXiv
2207.11620, behind the encoder / network / trainer / decoder API of the
CPU reference (/root/reference/pkg/src/neuralvol).  Host code is Python +
PyTorch (device memory, streams, torch.distributed); all compute is
hand-written CUDA in libnvol.so reached through the C ABI of include/nvol.h.
There is no CPU fallback: compute calls raise when the library or a CUDA
device is missing.
"""

__version__ = "0.1.0"

from . import _lib  # noqa: F401
from .errors import ConfigError, FormatError, MajorantViolation  # noqa: F401
