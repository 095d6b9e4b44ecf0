"""The C-ABI library loads without a GPU and exports every symbol that
include/lrqk_b200.h declares (no compute calls here)."""

import ctypes
import os
import re

import pytest

from paper_2510_23649_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "lrqk_b200.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(lrqk_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("lrqk_decode_step", "lrqk_decode_compress", "lrqk_score", "lrqk_select",
                 "lrqk_gather_misses", "lrqk_attention", "lrqk_prefill_factorize", "lrqk_seed_prompt"):
        assert must in names


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(_lib.LIB_PATH)
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_matches_header_layout():
    lib = _lib.load_library()
    assert lib.lrqk_abi_version() == 2
    assert lib.lrqk_sizeof_layer() == ctypes.sizeof(_lib.LayerStruct)
    assert lib.lrqk_sizeof_prefill() == ctypes.sizeof(_lib.PrefillStruct)
    assert set(_lib.SIGNATURES) >= set(declared_functions())


def test_buffer_sizes_for_north_star_layer():
    """Per-layer footprint at LLaMA-3-8B / 128K / r=32 / k=2048 (bf16)."""
    lib = _lib.load_library()
    s = _lib.LayerStruct()
    s.batch, s.n_q_heads, s.n_kv_heads, s.head_dim, s.dim_stride = 1, 32, 8, 128, 128
    s.rank, s.rank_stride, s.t_max, s.k_budget, s.lite_budget = 32, 32, 131072 + 256, 2048, 16
    s.s_cap, s.n_slots, s.cand_cap, s.dtype, s.policy, s.max_iter = 2064, 2065, 8192, _lib.BF16, _lib.SLOW_HBM, 2
    sizes = (ctypes.c_size_t * 64)()
    n = lib.lrqk_layer_buffer_bytes(ctypes.byref(s), sizes, 64)
    got = dict(zip(_lib.BUFFER_NAMES, sizes[:n]))
    assert got["proxy"] == 32 * (131072 + 256) * 32 * 2
    assert got["slow_k"] == 8 * (131072 + 256) * 128 * 2
    assert got["slot_k"] == 0  # HBM policy keeps no slots
    assert lib.lrqk_workspace_size(ctypes.byref(s)) == sum(sizes[:n])


def test_invalid_configuration_rejected():
    lib = _lib.load_library()
    s = _lib.LayerStruct()
    s.batch = 1
    s.n_q_heads, s.n_kv_heads = 3, 2  # not a GQA grouping
    sizes = (ctypes.c_size_t * 64)()
    assert lib.lrqk_layer_buffer_bytes(ctypes.byref(s), sizes, 64) == -1


def test_compute_entry_points_refuse_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(_lib.LibraryUnavailable):
        _lib.lib()
