"""ctypes binding of libttb.so (include/ttb.h). No torch types cross the ABI:
device pointers travel as integers and streams as cudaStream_t handles.

There is no CPU fallback: if the library is missing or CUDA is unavailable
every compute entry point raises.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

_HERE = Path(__file__).resolve().parent
# TTB_LIB_PATH: an alternative build of the same ABI (A/B timing in tools/)
LIB_PATH = Path(os.environ.get("TTB_LIB_PATH", str(_HERE / "libttb.so")))

TTB_OK = 0
TTB_EINVAL = -1
TTB_ERANGE = -2
TTB_EEMPTY = -3
TTB_EOFFSETS = -4
TTB_ENONFINITE = -5
TTB_ECUDA = -6
TTB_ESTATE = -7

ERRBIT_RANGE = 1
ERRBIT_EMPTY_BAG = 2
ERRBIT_OFFSETS = 4
ERRBIT_NONFINITE = 8
ERRBIT_PEER = 16

OPT_BWD_SPLIT = 1
OPT_FAST = 2
OPT_ALLOW_EMPTY = 3

# every symbol include/ttb.h declares (tests check the .so exports them all)
EXPORTS = [
    "ttb_abi_version", "ttb_strerror", "ttb_last_cuda_error", "ttb_launch_count", "ttb_workspace_bytes", "ttb_create",
    "ttb_destroy", "ttb_batched_workspace_bytes", "ttb_create_batched", "ttb_plan", "ttb_forward", "ttb_backward", "ttb_aggregate", "ttb_backward_sgd", "ttb_cores_modified", "ttb_sgd_update", "ttb_sgd_update_multi", "ttb_backward_adagrad", "ttb_adagrad_update", "ttb_dp_flag_words", "ttb_dp_exchange_update",
    "ttb_ipc_handle", "ttb_ipc_open", "ttb_ipc_close",
    "ttb_check_finite", "ttb_sgd_update_checked", "ttb_export_fast_plan", "ttb_plan_counts",
    "ttb_read_status", "ttb_status_word", "ttb_export_plan", "ttb_export_unique", "ttb_export_slots",
    "ttb_profile_enable", "ttb_profile_read", "ttb_set_option", "ttb_fma_peak",
    "ttb_count_frequencies", "ttb_rank_workspace_bytes", "ttb_rank_rows", "ttb_apply_bijection",
]


class TtbGeom(C.Structure):
    _fields_ = [("m", C.c_int64 * 3), ("n", C.c_int32 * 3), ("r", C.c_int32 * 4)]


class TtbSgdTensor(C.Structure):
    """ttb_sgd_tensor (include/ttb.h): one parameter of ttb_sgd_update_multi."""
    _fields_ = [("param", C.c_void_p), ("grad", C.c_void_p), ("velocity", C.c_void_p), ("n", C.c_int64)]


_vp = C.c_void_p
_i64 = C.c_int64
_int = C.c_int
_dbl = C.c_double

_PROTOS = {
    "ttb_abi_version": (_int, []),
    "ttb_strerror": (C.c_char_p, [_int]),
    "ttb_last_cuda_error": (C.c_char_p, []),
    "ttb_launch_count": (_i64, []),
    "ttb_workspace_bytes": (_int, [C.POINTER(TtbGeom), _i64, _i64, C.POINTER(C.c_size_t)]),
    "ttb_create": (_vp, [C.POINTER(TtbGeom), _i64, _i64, _vp, C.c_size_t, _vp]),
    "ttb_batched_workspace_bytes": (_int, [C.POINTER(TtbGeom), _int, _i64, _i64, C.POINTER(C.c_size_t)]),
    "ttb_create_batched": (_vp, [C.POINTER(TtbGeom), _int, _i64, _i64, _vp, C.c_size_t, _vp]),
    "ttb_destroy": (None, [_vp]),
    "ttb_plan": (_int, [_vp, _vp, _int, _vp, _i64, _i64, _vp]),
    "ttb_forward": (_int, [_vp, _vp, _vp, _vp, _vp, _vp]),
    "ttb_backward": (_int, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "ttb_aggregate": (_int, [_vp, _vp, _vp]),
    "ttb_backward_sgd": (_int, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _dbl, _dbl, _int, _vp]),
    "ttb_cores_modified": (_int, [_vp]),
    "ttb_sgd_update": (_int, [_vp, _vp, _vp, _i64, _dbl, _dbl, _vp]),
    "ttb_sgd_update_multi": (_int, [C.POINTER(TtbSgdTensor), _int, _dbl, _dbl, _vp]),
    "ttb_backward_adagrad": (_int, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _dbl, _dbl, _int, _vp]),
    "ttb_adagrad_update": (_int, [_vp, _vp, _vp, _i64, _dbl, _dbl, _vp, _vp]),
    "ttb_dp_flag_words": (C.c_size_t, [_int]),
    "ttb_dp_exchange_update": (_int, [_vp, _i64, _dbl, _dbl, _int, _vp, _vp, _int, _vp]),
    "ttb_ipc_handle": (_int, [_vp, _vp, C.POINTER(_i64)]),
    "ttb_ipc_open": (_int, [_vp, _i64, C.POINTER(_vp)]),
    "ttb_ipc_close": (_int, [_vp, _i64]),
    "ttb_check_finite": (_int, [_vp, _i64, _vp, _vp]),
    "ttb_sgd_update_checked": (_int, [_vp, _vp, _vp, _i64, _dbl, _dbl, _vp, _vp]),
    "ttb_read_status": (_int, [_vp, C.POINTER(_i64), _vp]),
    "ttb_status_word": (_vp, [_vp]),
    "ttb_export_plan": (_int, [_vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "ttb_export_unique": (_int, [_vp, _vp, _vp, _vp]),
    "ttb_plan_counts": (_int, [_vp, C.POINTER(_i64), _vp]),
    "ttb_export_fast_plan": (_int, [_vp, C.POINTER(_i64), _vp, _vp, _vp, _vp, _vp, _vp]),
    "ttb_export_slots": (_int, [_vp, _vp, _vp]),
    "ttb_profile_enable": (_int, [_vp, _int]),
    "ttb_profile_read": (_int, [_vp, _vp, _vp, _vp, _int, C.POINTER(_int)]),
    "ttb_set_option": (_int, [_vp, _int, _int]),
    "ttb_count_frequencies": (_int, [_vp, _i64, _i64, _vp, _vp, _vp]),
    "ttb_rank_workspace_bytes": (_int, [_i64, C.POINTER(C.c_size_t)]),
    "ttb_rank_rows": (_int, [_vp, _i64, _vp, _vp, _vp, C.c_size_t, _vp]),
    "ttb_apply_bijection": (_int, [_vp, _i64, _vp, _vp, _i64, _vp, _vp]),
    "ttb_fma_peak": (_int, [_vp, _int, _int, _vp]),
}

_lib = None


def load(path: str | os.PathLike | None = None):
    """Loads (once) and returns the CDLL with prototypes set. Raises if the
    library is absent — the product path has no fallback."""
    global _lib
    if _lib is not None:
        return _lib
    p = Path(path) if path else LIB_PATH
    if not p.exists():
        raise RuntimeError(
            f"{p} is missing: build the CUDA extension first "
            "(python -c 'import __graft_entry__ as g; g.build()')")
    lib = C.CDLL(str(p))
    for name, (res, args) in _PROTOS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


class TtbError(RuntimeError):
    pass


def check(code: int, what: str = "") -> None:
    """Maps a status code to the reference's exception types: data errors
    raise ValueError (as lookup.py / backward.py do), the rest RuntimeError."""
    if code == TTB_OK:
        return
    msg = load().ttb_strerror(code).decode()
    if what:
        msg = f"{what}: {msg}"
    if code in (TTB_EINVAL, TTB_ERANGE, TTB_EEMPTY, TTB_EOFFSETS, TTB_ENONFINITE):
        raise ValueError(msg)
    if code == TTB_ECUDA:
        msg = f"{msg} ({load().ttb_last_cuda_error().decode()})"
    raise TtbError(msg)


DP_MAX_PEERS = 8


class DpPeers(C.Structure):
    """ttb_dp_peers (include/ttb.h)."""
    _fields_ = [("rank", _int), ("world", _int), ("grad", _vp * DP_MAX_PEERS), ("param", _vp * DP_MAX_PEERS),
                ("flags", _vp * DP_MAX_PEERS)]


def errbits_to_exception(bits: int):
    if bits & ERRBIT_RANGE:
        return ValueError("bag index outside [0, rows)")
    if bits & ERRBIT_EMPTY_BAG:
        return ValueError("index bag must be a non-empty flat sequence")
    if bits & ERRBIT_OFFSETS:
        return ValueError("malformed bag offsets")
    if bits & ERRBIT_NONFINITE:
        return ValueError("non-finite gradient")
    if bits & ERRBIT_PEER:
        return RuntimeError("data-parallel exchange: a peer rank did not arrive")
    return None


def launch_count() -> int:
    return int(load().ttb_launch_count())
