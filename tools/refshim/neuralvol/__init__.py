"""Import shim: `neuralvol` (the reference package, /root/reference/pkg/src/neuralvol)
resolved to this repository's B200 package, so the reference's own test files run
against paper_2207_11620_b200 unmodified (SURVEY.md §8(b) drop-in evidence).

Every submodule the reference tests import is aliased to the package module of the
same name; `_kernels` (the reference's numba FFI) is served by ._kernels over the
C ABI.  Modules the package does not rebuild (service, image: out of the hot-path
scope) are simply absent, so the tests importing them fail at import and are
reported as such; _render_kernels exposes only the counter uniform the tests call.
"""
import importlib
import sys

__version__ = "0.1.0"

for _name in ("encoding", "network", "model", "trainer", "sampler", "volume", "fields", "macrocell",
              "render", "camera", "transfer", "errors", "estimator", "rng", "cli", "tracking"):
    _mod = importlib.import_module(f"paper_2207_11620_b200.{_name}")
    sys.modules[f"{__name__}.{_name}"] = _mod
    globals()[_name] = _mod
