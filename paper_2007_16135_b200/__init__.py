"""B200-native Time Warp Edit Distance (arXiv:2007.16135), sm_100a CUDA kernels.

Drop-in for the reference package's hot path (twedband / warpband):
``twed``, ``twed_batch`` (cuTWED-style north-star spellings, also accepting
the reference's ``lam=`` / ``symmetric=`` / list inputs), the
``paper_2007_16135_b200.warpband`` module with the reference bindings'
exact signatures, and device-resident ``twed_dev`` / ``twed_batch_dev``.
All compute runs in libtwb200.so; there is no CPU fallback.
"""

from .api import (
    band_solve,
    batch_matrix,
    lcs,
    mirror_upper_dev,
    prepare_series,
    twed,
    twed_batch,
    twed_batch_dev,
    twed_dev,
    twed_series,
)
from .core import InvalidInputError, TimeSeries, TwedParams
from ._lib import TwbError, device_count

__version__ = "0.2.0"

__all__ = [
    "InvalidInputError",
    "TimeSeries",
    "TwbError",
    "TwedParams",
    "band_solve",
    "batch_matrix",
    "device_count",
    "lcs",
    "mirror_upper_dev",
    "prepare_series",
    "twed",
    "twed_batch",
    "twed_batch_dev",
    "twed_dev",
    "twed_series",
    "__version__",
]
