"""ctypes binding of the C-ABI library ``librdist_b200.so`` (include/rdist_b200.h).

PyTorch is plumbing here: it owns device memory and the current CUDA stream;
every computation is a call into the sm_100a kernels of the shared library.
There is no CPU fallback: if the library or a CUDA device is missing, the
compute entry points raise :class:`NativeUnavailableError`.
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

import torch

_HERE = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("RDB_LIB_PATH") or _HERE / "librdist_b200.so")  # RDB_LIB_PATH: A/B builds (tools/)

RDB_ABI_VERSION = 6  # include/rdist_b200.h; load_library refuses a library built from another header
RDB_NB = 128
RDB_OK = 0
RDB_PIV_NONPOS = 1
RDB_PIV_NONFINITE = 2
RDB_BUILD_X = 0
RDB_BUILD_M = 1
RDB_CNT_NEGATIVE = 0
RDB_CNT_UNDERFLOW = 1
RDB_CNT_D8_RANGE = 2
RDB_NCOUNTERS = 3
RDB_D8_MAX = 254
RDB_D8_UNREACHABLE = 255
INT32_SENTINEL = 2147483647


class NativeUnavailableError(RuntimeError):
    """The CUDA library or a CUDA device is not available (no CPU fallback)."""


class NativeCallError(RuntimeError):
    """A C-ABI call returned an error status."""


class PivotInfo(ctypes.Structure):
    _fields_ = [("min_pivot", ctypes.c_double), ("min_index", ctypes.c_int32), ("flags", ctypes.c_int32)]


_i64 = ctypes.c_int64
_vp = ctypes.c_void_p
_dbl = ctypes.c_double
_int = ctypes.c_int
_sz = ctypes.c_size_t

# name -> (restype, argtypes); must match include/rdist_b200.h
SIGNATURES: dict[str, tuple[object, list[object]]] = {
    "rdb_strerror": (ctypes.c_char_p, [_int]),
    "rdb_abi_version": (_int, []),
    "rdb_last_cuda_error": (ctypes.c_char_p, []),
    "rdb_build_m": (_int, [_vp, _i64, _i64, _i64, _i64, _i64, _vp, _dbl, _int, _vp, _i64, _i64, _vp]),
    "rdb_build_m_bits": (_int, [_vp, _i64, _i64, _i64, _vp, _dbl, _vp, _i64, _i64, _vp]),
    "rdb_pad_identity": (_int, [_vp, _i64, _i64, _i64, _i64, _i64, _vp]),
    "rdb_matrix_stats": (_int, [_vp, _i64, _i64, _vp, _vp]),
    "rdb_invert_workspace_bytes": (_sz, [_i64, _i64]),
    "rdb_invert_batched_bits": (_int, [_vp, _i64, _i64, _i64, _i64, _vp, _i64, _vp, _vp, _vp]),
    "rdb_invert_batched": (_int, [_vp, _i64, _i64, _i64, _i64, _vp, _vp, _vp]),
    "rdb_invert": (_int, [_vp, _i64, _i64, _vp, _vp, _vp]),
    "rdb_gj_panel_inverse": (_int, [_vp, _i64, _vp, _int, _i64, _vp]),
    "rdb_gemm_local": (
        _int,
        [_vp, _i64, _vp, _i64, _vp, _i64, _i64, _i64, _i64, _i64, _i64, _i64, _int, _int, _i64, _vp],
    ),
    "rdb_invert_pivoted_workspace_bytes": (_sz, [_i64]),
    "rdb_invert_pivoted": (_int, [_vp, _i64, _i64, _vp, _vp, _vp]),
    "rdb_log_ceil": (
        _int,
        [_vp, _i64, _i64, _i64, _i64, _vp, _dbl, _vp, _vp, _vp, _i64, _i64, _vp, _i64, _vp, _vp],
    ),
    "rdb_log_ceil_block": (
        _int,
        [_vp, _i64, _i64, _i64, _i64, _i64, _vp, _dbl, _vp, _vp, _vp, _i64, _vp, _vp],
    ),
    "rdb_residual": (_int, [_vp, _i64, _vp, _i64, _i64, _vp, _vp]),
    "rdb_power_workspace_bytes": (_sz, [_i64]),
    "rdb_power_iteration": (_int, [_vp, _i64, _i64, _int, _dbl, _i64, _vp, _vp, _vp]),
    "rdb_count_edges": (_int, [_vp, _i64, _i64, _vp, _vp]),
    "rdb_next_hop_workspace_bytes": (_sz, [_i64, _i64, _i64]),
    "rdb_next_hop": (_int, [_vp, _i64, _vp, _i64, _i64, _i64, _vp, _i64, _vp, _i64, _vp, _vp]),
    "rdb_apsp_bits_batched": (_int, [_vp, _i64, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "rdb_log_ceil_d8": (_int, [_vp, _i64, _i64, _i64, _i64, _vp, _dbl, _vp, _i64, _i64, _vp, _vp]),
    "rdb_apsp_bits_batched_d8": (_int, [_vp, _i64, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "rdb_edges_to_bits": (_int, [_vp, _vp, _i64, _i64, _vp, _vp]),
    "rdb_bfs_workspace_bytes": (_sz, [_i64]),
    "rdb_pattern_bits": (_int, [_vp, _i64, _i64, _vp, _vp]),
    "rdb_bfs_apsp": (_int, [_vp, _i64, _vp, _vp, _i64, _vp, _vp, _vp]),
    "rdb_floyd_workspace_bytes": (_sz, [_i64]),
    "rdb_floyd_warshall": (_int, [_vp, _i64, _i64, _vp, _i64, _vp, _vp]),
    "rdb_global_accuracy": (_int, [_vp, _i64, _vp, _i64, _i64, _vp, _vp]),
    "rdb_local_accuracy": (
        _int,
        [_vp, _i64, _vp, _vp, _i64, _vp, _i64, _vp, _i64, _vp, _i64, _i64, _dbl, _vp, _vp, _vp],
    ),
}

_lib = None
_lock = threading.Lock()


def load_library(path: str | os.PathLike | None = None) -> ctypes.CDLL:
    """Load the shared library and declare every exported signature."""
    global _lib
    with _lock:
        if _lib is not None and path is None:
            return _lib
        p = Path(path) if path is not None else LIB_PATH
        if not p.exists():
            raise NativeUnavailableError(
                f"{p} not built; run `python -c 'import __graft_entry__ as g; g.build()'` or `make`"
            )
        lib = ctypes.CDLL(str(p))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.rdb_abi_version() != RDB_ABI_VERSION:
            raise NativeUnavailableError(f"{p}: ABI {lib.rdb_abi_version()} != {RDB_ABI_VERSION}; rebuild (`make`)")
        if path is None:
            _lib = lib
        return lib


def lib() -> ctypes.CDLL:
    return _lib if _lib is not None else load_library()


def device() -> torch.device:
    """The CUDA device the kernels run on; raises when there is none."""
    if not torch.cuda.is_available():
        raise NativeUnavailableError("a CUDA device is required (the B200 path has no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def stream_handle() -> int:
    return torch.cuda.current_stream().cuda_stream


def ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def check(rc: int, what: str) -> None:
    if rc != RDB_OK:
        msg = lib().rdb_strerror(rc).decode()
        if rc == 4:
            msg += f" [{lib().rdb_last_cuda_error().decode()}]"
        raise NativeCallError(f"{what} failed: {msg} (code {rc})")


def pad_to_nb(n: int) -> int:
    return (n + RDB_NB - 1) // RDB_NB * RDB_NB


def read_pivot_info(info: torch.Tensor) -> list[PivotInfo]:
    """info: uint8 device tensor holding `k` rdb_pivot_info records."""
    host = info.cpu().numpy().tobytes()
    k = len(host) // ctypes.sizeof(PivotInfo)
    return [PivotInfo.from_buffer_copy(host, i * ctypes.sizeof(PivotInfo)) for i in range(k)]


def pivot_info_tensor(k: int, dev: torch.device) -> torch.Tensor:
    return torch.zeros(k * ctypes.sizeof(PivotInfo), dtype=torch.uint8, device=dev)
