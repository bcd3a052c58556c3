"""ctypes binding of liblwb200.so (include/lw_b200.h).

The library is required: there is no CPU fallback behind the cuda backend. If
the .so is missing or fails to load, every device entry point raises
:class:`BackendUnavailable` naming the reason.
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "_lib" / "liblwb200.so"

LW_OK = 0
LW_E_INVALID_ARG = 10001
LW_E_UNSUPPORTED = 10002
LW_E_WORKSPACE = 10003
LW_E_NO_DEVICE = 10004
LW_E_FORMAT = 10005

LW_F32 = 0
LW_F64 = 1

LW_THREAD_MAPPED = 0
LW_MERGE_PATH = 1
LW_GROUP_MAPPED = 2

# every symbol include/lw_b200.h declares
EXPORTS = (
    "lw_error_string",
    "lw_abi_version",
    "lw_device_sm_count",
    "lw_auto_lanes",
    "lw_merge_path_partition",
    "lw_group_plan_prefix",
    "lw_spmv_thread_mapped",
    "lw_spmv_work_oriented_workspace",
    "lw_spmv_work_oriented",
    "lw_spmv_work_oriented_phases",
    "lw_spmv_work_oriented_peers",
    "lw_spmv_work_oriented_peers_hotx",
    "lw_hotx_build_workspace",
    "lw_hotx_build",
    "lw_spmv_work_oriented_hotx_workspace",
    "lw_spmv_work_oriented_hotx",
    "lw_spmv_work_oriented_hotx_phases",
    "lw_debug_lane_atom_counts",
    "lw_debug_atom_tiles",
    "lw_norm_workspace",
    "lw_vector_norm",
    "lw_vector_scale",
    "lw_spmv_group_mapped",
    "lw_spmv_workspace",
    "lw_spmv",
    "lw_spmv_host",
    "lw_spmm_auto_lanes",
    "lw_spmm_workspace",
    "lw_spmm_thread_mapped",
    "lw_spmm_work_oriented",
    "lw_spmm_group_mapped",
    "lw_spmm",
    "lw_frontier_workspace",
    "lw_frontier_compact",
    "lw_sssp_pass",
    "lw_bfs_pass",
    "lw_sssp",
    "lw_bfs",
    "lw_mm_parse_header",
    "lw_mm_parse_entries",
    "lw_coo_to_csr_host",
    "lw_rmat_keys",
    "lw_hash_values",
    "lw_uniform_keys",
    "lw_csr_permute",
)


class BackendUnavailable(RuntimeError):
    """The CUDA library or a CUDA device is not available."""


class LwCsr(ctypes.Structure):
    _fields_ = [
        ("rows", ctypes.c_int64),
        ("cols", ctypes.c_int64),
        ("nnz", ctypes.c_int64),
        ("row_offsets", ctypes.c_void_p),
        ("col_indices", ctypes.c_void_p),
        ("values", ctypes.c_void_p),
        ("offset_bits", ctypes.c_int32),
        ("dtype", ctypes.c_int32),
    ]


class LwProbe(ctypes.Structure):
    _fields_ = [
        ("lane_atoms", ctypes.c_void_p),
        ("atom_lane", ctypes.c_void_p),
        ("atom_tile", ctypes.c_void_p),
        ("atom_visits", ctypes.c_void_p),
    ]


class LwMmHeader(ctypes.Structure):
    _fields_ = [
        ("rows", ctypes.c_int64),
        ("cols", ctypes.c_int64),
        ("entries", ctypes.c_int64),
        ("field", ctypes.c_int32),
        ("symmetric", ctypes.c_int32),
        ("data_offset", ctypes.c_int64),
    ]


_lock = threading.Lock()
_lib = None
_load_error: str | None = None

_i64 = ctypes.c_int64
_u64 = ctypes.c_uint64
_i32 = ctypes.c_int32
_u32 = ctypes.c_uint32
_vp = ctypes.c_void_p
_sz = ctypes.c_size_t
_up = ctypes.c_size_t  # uintptr_t stream
_csr_p = ctypes.POINTER(LwCsr)
_probe_p = ctypes.POINTER(LwProbe)

_SIGNATURES = {
    "lw_error_string": (ctypes.c_char_p, [ctypes.c_int]),
    "lw_abi_version": (ctypes.c_int, []),
    "lw_device_sm_count": (ctypes.c_int, [ctypes.POINTER(ctypes.c_int)]),
    "lw_auto_lanes": (ctypes.c_int, [ctypes.c_int, _i64, _i64, _i64, _i64, ctypes.POINTER(_i64)]),
    "lw_merge_path_partition": (ctypes.c_int, [_i64, _i64, _vp, _i32, _i64, _vp, _up]),
    "lw_group_plan_prefix": (ctypes.c_int, [_i64, _vp, _i32, _i64, _vp, _up]),
    "lw_spmv_thread_mapped": (ctypes.c_int, [_csr_p, _vp, _vp, _i64, _probe_p, _up]),
    "lw_spmv_work_oriented_workspace": (_sz, [_i64, _i64, _i64, _i32]),
    "lw_spmv_work_oriented": (ctypes.c_int, [_csr_p, _vp, _vp, _i64, _vp, _sz, _probe_p, _up]),
    "lw_spmv_work_oriented_phases": (ctypes.c_int, [_csr_p, _vp, _vp, _i64, _vp, _sz, _u32, _up]),
    "lw_spmv_work_oriented_peers": (ctypes.c_int, [_csr_p, _vp, _vp, _i64, _vp, _sz, _i32, _vp, _u64,
                                                   _i64, _up]),
    "lw_spmv_work_oriented_peers_hotx": (ctypes.c_int, [_csr_p, _vp, _i32, _vp, _vp, _i64, _vp, _sz, _i32,
                                                        _vp, _u64, _i64, _up]),
    "lw_hotx_build_workspace": (_sz, [_i64]),
    "lw_hotx_build": (ctypes.c_int, [_csr_p, _i32, _vp, _vp, ctypes.POINTER(_i32), _vp, _sz, _up]),
    "lw_spmv_work_oriented_hotx_workspace": (_sz, [_i64, _i64, _i64, _i32, _i32]),
    "lw_spmv_work_oriented_hotx": (ctypes.c_int, [_csr_p, _vp, _i32, _vp, _vp, _i64, _vp, _sz, _up]),
    "lw_spmv_work_oriented_hotx_phases": (ctypes.c_int, [_csr_p, _vp, _i32, _vp, _vp, _i64, _vp, _sz,
                                                         _u32, _up]),
    "lw_debug_lane_atom_counts": (ctypes.c_int, [ctypes.c_int, _csr_p, _vp, _vp, _i64, _i64, _i64, _vp, _vp, _sz,
                                                 _up]),
    "lw_debug_atom_tiles": (ctypes.c_int, [ctypes.c_int, _csr_p, _vp, _vp, _i64, _i64, _i64, _vp, _vp, _vp, _sz,
                                           _up]),
    "lw_norm_workspace": (_sz, [_i64]),
    "lw_vector_norm": (ctypes.c_int, [_vp, _i64, _i32, _vp, _sz, _vp, _up]),
    "lw_vector_scale": (ctypes.c_int, [_vp, _i64, _i32, _vp, _vp, _up]),
    "lw_spmv_group_mapped": (ctypes.c_int, [_csr_p, _vp, _vp, _i64, _i64, _i64, _probe_p, _up]),
    "lw_spmv_workspace": (_sz, [ctypes.c_int, _i64, _i64, _i64, _i32]),
    "lw_spmv": (ctypes.c_int, [ctypes.c_int, _csr_p, _vp, _vp, _i64, _i64, _i64, _vp, _sz, _up]),
    "lw_spmv_host": (ctypes.c_int, [ctypes.c_int, _csr_p, _vp, _vp, _i64, _i64, _i64, _up]),
    "lw_spmm_auto_lanes": (ctypes.c_int, [ctypes.c_int, _i64, _i64, _i64, _i64, _i64,
                                          ctypes.POINTER(_i64)]),
    "lw_spmm_workspace": (_sz, [ctypes.c_int, _i64, _i64, _i64, _i64, _i32]),
    "lw_spmm_thread_mapped": (ctypes.c_int, [_csr_p, _vp, _vp, _i64, _i64, _up]),
    "lw_spmm_work_oriented": (ctypes.c_int, [_csr_p, _vp, _vp, _i64, _i64, _vp, _sz, _up]),
    "lw_spmm_group_mapped": (ctypes.c_int, [_csr_p, _vp, _vp, _i64, _i64, _i64, _i64, _up]),
    "lw_spmm": (ctypes.c_int, [ctypes.c_int, _csr_p, _vp, _vp, _i64, _i64, _i64, _i64, _vp, _sz,
                               _up]),
    "lw_frontier_workspace": (_sz, [_i64]),
    "lw_frontier_compact": (ctypes.c_int, [_vp, _i64, _vp, _vp, _vp, _sz, _up]),
    "lw_sssp_pass": (ctypes.c_int, [_csr_p, _vp, _i64, _vp, _vp, ctypes.c_int, _i64, _i64, _i64,
                                    _vp, _sz, _up]),
    "lw_bfs_pass": (ctypes.c_int, [_csr_p, _vp, _i64, _vp, _i64, _vp, ctypes.c_int, _i64, _i64,
                                   _i64, _vp, _sz, _up]),
    "lw_sssp": (ctypes.c_int, [_csr_p, _i64, _vp, ctypes.c_int, _i64, _i64, _i64, _vp, _sz,
                               ctypes.POINTER(_i64), _up]),
    "lw_bfs": (ctypes.c_int, [_csr_p, _i64, _vp, ctypes.c_int, _i64, _i64, _i64, _vp, _sz,
                              ctypes.POINTER(_i64), _up]),
    "lw_mm_parse_header": (ctypes.c_int, [ctypes.c_char_p, _sz, ctypes.POINTER(LwMmHeader),
                                          ctypes.c_char_p, _sz]),
    "lw_mm_parse_entries": (ctypes.c_int, [ctypes.c_char_p, _sz, ctypes.POINTER(LwMmHeader), _vp,
                                           _vp, _vp, _i64, ctypes.POINTER(_i64), _i32,
                                           ctypes.c_char_p, _sz]),
    "lw_coo_to_csr_host": (ctypes.c_int, [_i64, _i64, _i64, _vp, _vp, _vp, _vp, _vp, _vp,
                                          ctypes.POINTER(_i64), _i32]),
    "lw_rmat_keys": (ctypes.c_int, [_i32, _i64, _i64, _u32, _u32, _u32, _u64, _vp, _up]),
    "lw_hash_values": (ctypes.c_int, [_vp, _i64, _u64, _i32, _vp, _up]),
    "lw_uniform_keys": (ctypes.c_int, [_i64, _i64, _i64, _u64, _vp, _up]),
    "lw_csr_permute": (ctypes.c_int, [_csr_p, _vp, _vp, _vp, _vp, _vp, _up]),
}


def load(path: Path | str | None = None):
    """Load (once) and return the ctypes library; raises BackendUnavailable."""
    global _lib, _load_error
    with _lock:
        if _lib is not None:
            return _lib
        p = Path(path) if path else Path(os.environ.get("LWB200_LIB", LIB_PATH))
        if not p.exists():
            _load_error = f"{p} not built (run __graft_entry__.build() or python -m paper_2301_04792_b200._build)"
            raise BackendUnavailable(_load_error)
        try:
            lib = ctypes.CDLL(str(p))
        except OSError as exc:  # pragma: no cover - depends on the box
            _load_error = f"cannot load {p}: {exc}"
            raise BackendUnavailable(_load_error) from exc
        variant = "LWB200_LIB" in os.environ and not path   # A/B builds may predate new entries
        for name, (res, args) in _SIGNATURES.items():
            if variant and not hasattr(lib, name):
                continue
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def error_string(code: int) -> str:
    return load().lw_error_string(code).decode()


def check(code: int, what: str) -> None:
    """Map a C-ABI return code to the reference's exception types."""
    if code == LW_OK:
        return
    msg = f"{what}: {error_string(code)} (code {code})"
    if code == LW_E_INVALID_ARG:
        raise ValueError(msg)
    if code == LW_E_NO_DEVICE:
        raise BackendUnavailable(msg)
    raise RuntimeError(msg)


def sm_count() -> int:
    n = ctypes.c_int(0)
    check(load().lw_device_sm_count(ctypes.byref(n)), "lw_device_sm_count")
    return n.value


def auto_lanes(schedule: int, rows: int, nnz: int, group_size: int = 32,
               tiles_per_block: int = 32) -> int:
    out = _i64(0)
    check(load().lw_auto_lanes(schedule, rows, nnz, group_size, tiles_per_block,
                               ctypes.byref(out)), "lw_auto_lanes")
    return out.value
