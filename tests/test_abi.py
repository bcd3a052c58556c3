"""The C-ABI library: loads without a GPU, exports every symbol the header
declares, and rejects bad arguments with LW_E_* codes (no kernel launches)."""

import ctypes
import re
from pathlib import Path

import pytest

from paper_2301_04792_b200 import _build, _lib

HEADER = Path(__file__).resolve().parents[1] / "include" / "lw_b200.h"


def declared_symbols():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(lw_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    _build.build()
    return _lib.load()


def test_header_and_binding_agree():
    assert declared_symbols() == sorted(_lib.EXPORTS)


def test_every_declared_symbol_is_exported(lib):
    for name in declared_symbols():
        assert hasattr(lib, name), name


def test_library_is_sm100a_only():
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib.LIB_PATH)], capture_output=True,
                         text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    arches = set(re.findall(r"sm_\d+a?", out.stdout))
    assert arches == {"sm_100a"}, arches


def test_error_strings_and_version(lib):
    assert lib.lw_abi_version() == 1
    assert b"invalid" in lib.lw_error_string(_lib.LW_E_INVALID_ARG)
    assert b"workspace" in lib.lw_error_string(_lib.LW_E_WORKSPACE)
    assert lib.lw_error_string(0) == b"success"


def test_invalid_arguments_are_rejected_without_a_device(lib):
    out = ctypes.c_int64(0)
    assert lib.lw_auto_lanes(7, 10, 10, 32, 32, ctypes.byref(out)) == _lib.LW_E_INVALID_ARG
    assert lib.lw_auto_lanes(2, 10, 10, 0, 32, ctypes.byref(out)) == _lib.LW_E_INVALID_ARG
    assert lib.lw_auto_lanes(1, -1, 10, 32, 32, ctypes.byref(out)) == _lib.LW_E_INVALID_ARG
    assert lib.lw_auto_lanes(1, 10, 0, 32, 32, ctypes.byref(out)) == 0
    assert out.value == 1  # one 2040-item chunk (CTA) covers 10 rows
    a = _lib.LwCsr()
    a.rows, a.cols, a.nnz, a.offset_bits, a.dtype = 2, 2, 2, 16, 0
    assert lib.lw_spmv_thread_mapped(ctypes.byref(a), None, None, 0, None, 0) == _lib.LW_E_INVALID_ARG
    a.offset_bits, a.dtype = 32, 5
    assert lib.lw_spmv(0, ctypes.byref(a), None, None, 0, 32, 32, None, 0, 0) == _lib.LW_E_INVALID_ARG
    a.dtype = 0
    assert lib.lw_spmv(9, ctypes.byref(a), None, None, 0, 32, 32, None, 0, 0) == _lib.LW_E_INVALID_ARG
    assert lib.lw_merge_path_partition(1, 1, None, 32, 0, None, 0) == _lib.LW_E_INVALID_ARG
    assert lib.lw_rmat_keys(0, 0, 10, 1, 2, 3, 1, None, 0) == _lib.LW_E_INVALID_ARG
    assert lib.lw_spmv_work_oriented_workspace(10, 10, 0, 0) > 0


def test_workspace_query_scales_with_lanes(lib):
    small = lib.lw_spmv_work_oriented_workspace(1000, 100000, 64, 0)
    auto = lib.lw_spmv_work_oriented_workspace(1000, 100000, 0, 0)
    assert small > 0 and auto > 0
    assert lib.lw_spmv_workspace(0, 1000, 100000, 0, 0) == 0


def test_hotx_entry_points_validate_without_a_device(lib):
    """The hot-x packing entries reject bad shapes before touching a device."""
    a = _lib.LwCsr()
    a.rows, a.cols, a.nnz, a.offset_bits, a.dtype = 4, 4, 4, 32, _lib.LW_F32
    n = ctypes.c_int32(0)
    # slot cap above the one-CTA sort, negative cap, missing output count
    assert lib.lw_hotx_build(ctypes.byref(a), 32769, None, None, ctypes.byref(n), None, 0, 0) \
        == _lib.LW_E_INVALID_ARG
    assert lib.lw_hotx_build(ctypes.byref(a), -1, None, None, ctypes.byref(n), None, 0, 0) \
        == _lib.LW_E_INVALID_ARG
    assert lib.lw_hotx_build(ctypes.byref(a), 16, None, None, None, None, 0, 0) == _lib.LW_E_INVALID_ARG
    # packed SpMV: missing y / x, negative lanes
    assert lib.lw_spmv_work_oriented_hotx(ctypes.byref(a), None, 0, None, None, 0, None, 0, 0) \
        == _lib.LW_E_INVALID_ARG
    # workspace grows with the hot slots and covers at least one slot
    base = lib.lw_spmv_work_oriented_workspace(1000, 100000, 0, _lib.LW_F32)
    w0 = lib.lw_spmv_work_oriented_hotx_workspace(1000, 100000, 0, 0, _lib.LW_F32)
    w1 = lib.lw_spmv_work_oriented_hotx_workspace(1000, 100000, 0, 12288, _lib.LW_F32)
    assert base < w0 < w1 and w1 - base >= 12288 * 4
    assert lib.lw_hotx_build_workspace(1 << 20) >= (1 << 20) * 4
