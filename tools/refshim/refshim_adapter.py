"""pytest plugin for running the reference's test files against the B200 package
(tools/run_reference_tests.py): the reference compares results with numpy
(np.testing, np.asarray, ...), and the package hands out CUDA tensors where the
reference hands out numpy arrays.  The single adapter: numpy may read a CUDA tensor
(a device-to-host copy, like any other D2H).  Nothing else is patched; a test that
relies on other ndarray-only behaviour fails and is reported as such."""
import torch

_orig = torch.Tensor.__array__


def _array(self, dtype=None, copy=None):
    if self.is_cuda:
        a = self.detach().cpu().numpy()
        return a.astype(dtype, copy=False) if dtype is not None else a
    return _orig(self, dtype) if dtype is not None else _orig(self)


torch.Tensor.__array__ = _array
