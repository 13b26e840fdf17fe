"""B200-native execution path for tensorsel's convolution family
(arXiv 2512.02371, "Pushing Tensor Accelerators Beyond MatMul").

Public modules:
  layout     — the reference ``tensorsel.layout`` API (host + device builders)
  axis       — device-resident banded weight matrices (the weight builder)
  pipelines  — resample / filter / denoise on planar CUDA images
  partition  — frame / row-band sharding across the GPUs of one box
"""

__version__ = "0.1.0"

from . import errors, filters, layout  # noqa: F401  (import-safe without a GPU)
