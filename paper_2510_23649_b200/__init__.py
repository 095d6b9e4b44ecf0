"""B200-native LRQK decode-time sparse-attention path (arXiv 2510.23649).

Drop-in for the reference package's prefill / decode / cache-manager /
attention API (ref: pkg/src/lrqk/__init__.py:10-82), computed by hand-written
sm_100a CUDA kernels behind a C-ABI (include/lrqk_b200.h).  There is no CPU
fallback: without the library or a CUDA device every compute call raises
LibraryUnavailable.
"""

from .errors import CorruptTraceError, NonFiniteError, SolveFailedError, UnsupportedVersionError
from ._lib import LibraryUnavailable, load_library
from .engine import Engine, LayerShape, LayerState, prefill_factorize_device

__version__ = "0.1.0"
