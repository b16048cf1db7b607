"""The C-ABI library loads and exports every entry point include/slp_b200.h
declares (no device calls: runs without a GPU)."""

import ctypes
import os
import re

from paper_1805_01407_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    with open(os.path.join(ROOT, "include", "slp_b200.h")) as f:
        text = f.read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(slp_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_expected_surface():
    names = declared_functions()
    for must in ("slp_fill", "slp_fused", "slp_init_substreams", "slp_jump_states", "slp_char_poly",
                 "slp_jump_poly", "slp_host_jump", "slp_generator_id"):
        assert must in names


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(_native.LIB_PATH)
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_covers_header():
    assert set(declared_functions()) == set(_native.SIGNATURES)
    L = _native.lib()
    assert b"sm_100a" in L.slp_build_info()
    assert L.slp_status_str(_native.SLP_ERR_ZERO_STATE)


def test_device_entry_points_reject_bad_arguments_without_touching_the_gpu():
    L = _native.lib()
    # unknown generator / null pointers are rejected before any CUDA call
    assert L.slp_fill(999, None, None, 0, 0, 0, 0, 0, None, 0, None) == _native.SLP_ERR_UNKNOWN_GENERATOR
    assert L.slp_fill(8, None, None, 4, 4, 4, 0, 0, None, 4, None) == _native.SLP_ERR_INVALID
    assert L.slp_fill(8, None, None, 0, 0, 4, 0, 0, None, 4, None) == _native.SLP_OK  # nothing to do
    assert L.slp_fused(8, None, None, 0, 0, 0, 1, None, None, 0, None) == _native.SLP_ERR_INVALID
    assert L.slp_init_substreams(8, None, 1, None, 0, None, 1, 1, None) == _native.SLP_ERR_INVALID
    zero = (ctypes.c_uint64 * 4)()
    assert L.slp_jump_states(8, zero, 4, ctypes.c_void_p(16), 4, ctypes.c_void_p(16), 4, 4, None) \
        == _native.SLP_ERR_ZERO_STATE


def test_more_entry_points_reject_bad_arguments_without_touching_the_gpu():
    L = _native.lib()
    E = _native
    one = (ctypes.c_uint64 * 1)(1)
    # segment split: unknown generator, nothing to do, null pointers, too many segments
    assert L.slp_split_substreams(999, None, 1, 1, one, 1, 2, None, 2, None) == E.SLP_ERR_UNKNOWN_GENERATOR
    assert L.slp_split_substreams(8, None, 1, 0, one, 1, 2, None, 2, None) == E.SLP_OK
    assert L.slp_split_substreams(8, None, 1, 1, one, 1, 2, None, 2, None) == E.SLP_ERR_INVALID
    assert L.slp_split_substreams(8, ctypes.c_void_p(16), 1, 1, one, 1, (1 << 20) + 1, ctypes.c_void_p(16),
                                  (1 << 20) + 1, None) == E.SLP_ERR_INVALID
    assert L.slp_split_substreams(8, ctypes.c_void_p(16), 1, 1, one, 1, 4, ctypes.c_void_p(16), 3, None) \
        == E.SLP_ERR_INVALID  # ld_seg < n * J
    # one LanedStream superbatch
    assert L.slp_laned_fill(999, None, 1, 1, 0, None, None, None) == E.SLP_ERR_UNKNOWN_GENERATOR
    assert L.slp_laned_fill(8, None, 0, 4, 0, None, None, None) == E.SLP_OK
    assert L.slp_laned_fill(8, None, 4, 4, 0, None, None, None) == E.SLP_ERR_INVALID
    # store + checksum: result / workspace required
    assert L.slp_fill_checksum(999, None, None, 0, 0, 0, 0, None, 0, None, None, 0, None) \
        == E.SLP_ERR_UNKNOWN_GENERATOR
    assert L.slp_fill_checksum(8, None, None, 4, 4, 4, 0, None, 4, None, None, 0, None) == E.SLP_ERR_INVALID
    # HWD counting: k out of range, split on a 32-bit generator, inconsistent range
    cs = (ctypes.c_uint64 * 4)()
    assert L.slp_hwd_count(8, ctypes.c_void_p(16), 1, 1, 1, 1, 0, 0, 0, 0, 64, 0, 0, cs, cs, None, None) \
        == E.SLP_ERR_INVALID
    w32 = L.slp_generator_id(b"xoshiro128starstar")
    assert w32 >= 0
    assert L.slp_hwd_count(w32, ctypes.c_void_p(16), 1, 1, 1, 1, 0, 0, 2, 0, 32, 0, 1, cs, cs, None, None) \
        == E.SLP_ERR_INVALID
    assert L.slp_hwd_count(8, ctypes.c_void_p(16), 1, 2, 10, 5, 0, 0, 2, 0, 64, 0, 0, cs, cs, None, None) \
        == E.SLP_ERR_INVALID  # total <= (nthreads - 1) * tseg


def test_split_factor_is_host_only_and_follows_the_wave_rule():
    """slp_split_factor (no device call): 1 from 2^15 substreams up or for
    rows too short to split; else a power of two: segments >= 512 outputs up
    to half a wave (2^14 segments), >= 2048 beyond, n*J <= 2^18."""
    L = _native.lib()
    g = L.slp_generator_id(b"xoshiro256starstar")
    assert L.slp_split_factor(999, 1, 1 << 20) == _native.SLP_ERR_UNKNOWN_GENERATOR
    assert L.slp_split_factor(g, 1 << 15, 1 << 20) == 1
    assert L.slp_split_factor(g, 1000, 1023) == 1
    for n, T in [(1, 1 << 28), (16, 1 << 24), (1000, 1 << 18), (3, 3 << 16), (4096, 4096), (8192, 2048)]:
        J = L.slp_split_factor(g, n, T)
        assert J > 1 and J & (J - 1) == 0 and T % J == 0 and T // J >= 512 and n * J <= 1 << 18
        assert T // J >= 2048 or n * J <= 1 << 14
    assert L.slp_split_factor(g, 4096, 4096) == 4 and L.slp_split_factor(g, 1, 1 << 28) == 1 << 17
    big = L.slp_generator_id(b"xoroshiro1024starstar")
    assert (1 << 20) // L.slp_split_factor(big, 1, 1 << 20) >= 2 * 1024  # >= 2 outputs per state bit
    assert (1 << 28) // L.slp_split_factor(big, 1, 1 << 28) >= 8 * 1024  # long rows: >= 8 per state bit


def test_fill_pace_knob_is_host_only():
    """slp_set_fill_pace: query with a negative value, set, restore (no device call)."""
    from paper_1805_01407_b200 import device as D

    L = _native.lib()
    cur = L.slp_set_fill_pace(-1)
    assert cur >= 0
    assert L.slp_set_fill_pace(1234) == cur
    assert D.set_fill_pace(None) == 1234
    assert D.set_fill_pace(cur) == 1234
    assert L.slp_set_fill_pace(-1) == cur
