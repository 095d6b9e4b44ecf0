"""B200-native LRQK decode-time sparse-attention path (arXiv 2510.23649).

Drop-in for the reference package's prefill / decode / cache-manager /
attention API (ref: pkg/src/lrqk/__init__.py:10-82): the same names are
re-exported flat from this package, computed by hand-written sm_100a CUDA
kernels behind a C-ABI (include/lrqk_b200.h).  The batched multi-layer
engine (`Engine`, `LayerState`) is the throughput path.  There is no CPU
fallback: without the library or a CUDA device every compute call raises
LibraryUnavailable.
"""

from .errors import CorruptTraceError, NonFiniteError, SolveFailedError, UnsupportedVersionError
from ._lib import LibraryUnavailable, load_library
from .engine import Engine, LayerShape, LayerState, prefill_factorize_device
from .api import (
    AttentionResult,
    CacheStats,
    CompressedToken,
    DecodeConfig,
    DecodeSession,
    DecodeWorkspace,
    ImportanceScores,
    InitStrategy,
    LowRankFactors,
    PrefillConfig,
    PrefillRun,
    SelectionSet,
    SessionConfig,
    SimulationResult,
    StepReport,
    TieredKVCache,
    TokenStep,
    append_token,
    as_matrix,
    as_row,
    decode_compress,
    exact_attention,
    exact_topk,
    factor_residuals,
    fetch_and_merge,
    fro_norm_sq,
    gram,
    importance_scores,
    init_factors,
    khat_initial_guess,
    lagrangian_value,
    miss_rate,
    prefill_factorize,
    prefill_run,
    proxy_scores,
    run_simulation,
    select_active,
    selection_recall,
    solve_spd,
    summarize,
    topk_indices,
    update_AK,
    update_AQ,
    update_B,
    update_khat,
    update_projections,
    update_qhat,
    write_report_csv,
    write_stats_csv,
)

__version__ = "0.1.0"
