"""pytest plugin for running the reference's test files against the B200 package
(tools/run_reference_tests.py).  The reference hands out numpy arrays where the package
hands out CUDA tensors, and its tests use numpy idioms on them.  The adapter maps exactly
four idioms onto torch ("a thin adapter that maps these idioms onto torch
tensors"), nothing else:

  1. numpy reads a CUDA tensor (np.asarray / np.testing / ufuncs): a device-to-host copy;
  2. in-place writes of numpy arrays or lists into a CUDA tensor (`t[...] = ndarray`):
     converted to a tensor of t's dtype on t's device first;
  3. `t.copy()` (ndarray.copy) returns `t.clone()`;
  4. `t.astype(dtype)` returns the converted host array.

A test relying on any other ndarray-only behaviour (`.size` as an attribute, numpy dtype
objects, ...) fails and is reported as such.
"""
import numpy as np
import torch

_orig_array = torch.Tensor.__array__
_orig_setitem = torch.Tensor.__setitem__


def _array(self, dtype=None, copy=None):
    if self.is_cuda:
        a = self.detach().cpu().numpy()
        return a.astype(dtype, copy=False) if dtype is not None else a
    return _orig_array(self, dtype) if dtype is not None else _orig_array(self)


def _setitem(self, key, value):
    if self.is_cuda and isinstance(value, (np.ndarray, list, tuple, np.generic)):
        value = torch.as_tensor(np.asarray(value), dtype=self.dtype).to(self.device)
    return _orig_setitem(self, key, value)


torch.Tensor.__array__ = _array
torch.Tensor.__setitem__ = _setitem
torch.Tensor.copy = lambda self: self.clone()
# 4. `t.astype(dtype)` (ndarray.astype) returns the host array converted, as numpy would
torch.Tensor.astype = lambda self, dtype, copy=True: np.asarray(self).astype(dtype)
