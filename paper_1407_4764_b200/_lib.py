"""ctypes binding of ``libotf_b200.so`` (the C ABI in include/otf_b200.h).

There is no fallback: if the library is missing or no CUDA device is visible, every entry
point raises ``RetrievalError`` — the product path is the sm_100a kernels or nothing.
ctypes releases the GIL for the duration of each foreign call, so the ranker and trainer
threads of a live session (session.py:295-359 in the reference) overlap on the GPU.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

import numpy as np

from .errors import (
    ConfigError,
    CorruptionError,
    DegenerateInputError,
    EmptyStoreError,
    FormatError,
    InsufficientDataError,
    NotReadyError,
    RetrievalError,
)

LIB_PATH = Path(__file__).resolve().parent / "libotf_b200.so"

OK = 0
MEM_HOST, MEM_DEVICE = 0, 1
KIND_DENSE, KIND_PQ, KIND_BINARY = 0, 1, 2
F32, F64 = 0, 1

_ERRORS = {
    1: ConfigError,
    2: NotReadyError,
    3: InsufficientDataError,
    4: CorruptionError,
    5: EmptyStoreError,
    6: RetrievalError,
    7: RetrievalError,
    8: FormatError,
    9: DegenerateInputError,
    10: OSError,
}

_vp, _i64, _i32, _int, _dbl = C.c_void_p, C.c_int64, C.c_int32, C.c_int, C.c_double
_P = C.POINTER

# name -> argtypes (all return int unless listed in _RESTYPE)
SIGNATURES: dict[str, list] = {
    "otf_last_error": [],
    "otf_abi_version": [],
    "otf_device_count": [_P(_int)],
    "otf_set_reserved_sms": [_int, _i32],
    "otf_kernel_names": [],
    "otf_launch_count": [],
    "otf_repo_create_dense": [_int, _vp, _i64, _i32, _vp, _i64, _int, _int, _P(_vp)],
    "otf_repo_create_pq": [_int, _vp, _i64, _vp, _i32, _i32, _i32, _vp, _i64, _int, _int, _P(_vp)],
    "otf_repo_create_binary": [_int, _vp, _i64, _i32, _vp, _i64, _int, _int, _P(_vp)],
    "otf_repo_subset": [_vp, _vp, _i64, _P(_vp)],
    "otf_repo_destroy": [_vp],
    "otf_repo_load_dense": [_int, C.c_char_p, _int, _P(_vp)],
    "otf_repo_load_pq": [_int, C.c_char_p, _vp, _i32, _i32, _i32, _vp, _P(_vp)],
    "otf_repo_load_binary": [_int, C.c_char_p, _i32, _vp, _P(_vp), _P(_i32)],
    "otf_file_read_bench": [C.c_char_p, _i64, _P(_dbl), _P(_i64)],
    "otf_repo_info": [_vp, _P(_i32), _P(_i64), _P(_i32), _P(_i64), _P(_i32)],
    "otf_repo_score": [_vp, _vp, _vp, _int, _vp],
    "otf_repo_time_rank_scan": [_vp, _vp, _i64, _vp, _vp],
    "otf_repo_cut_fallbacks": [_vp, _P(_i64)],
    "otf_repo_rank": [_vp, _vp, _i64, _vp, _vp, _vp, _P(_i64), _int, _vp],
    "otf_repo_rank_graph": [_vp, _vp, _i64, _vp, _vp, _vp, _vp],
    "otf_repo_score_many": [_vp, _vp, _i32, _vp, _int, _vp],
    "otf_repo_rank_many": [_vp, _vp, _i32, _i64, _vp, _vp, _P(_i64), _int, _vp],
    "otf_score_dense": [_int, _vp, _i64, _i32, _vp, _vp, _int, _vp],
    "otf_pq_build_lut": [_int, _vp, _i32, _i32, _i32, _vp, _vp, _int, _vp],
    "otf_pq_score_codes": [_int, _vp, _i32, _i32, _vp, _i64, _vp, _int, _vp],
    "otf_score_binary": [_int, _vp, _i64, _i32, _vp, _vp, _int, _vp],
    "otf_unpack_bits": [_int, _vp, _i64, _i32, _vp, _int, _vp],
    "otf_binarize": [_int, _vp, _vp, _i32, _i32, _vp, _i64, _vp, _int, _vp],
    "otf_hamming": [_int, _vp, _vp, _i64, _i32, _vp, _int, _vp],
    "otf_top_k": [_int, _vp, _i32, _i64, _vp, _i64, _vp, _vp, _vp, _P(_i64), _int, _vp],
    "otf_pegasos_update": [_int, _vp, _i32, _vp, _i32, _i64, _vp, _i32, _i64, _vp, _vp, _i32,
                           _dbl, _dbl, _int, _dbl, _vp],
    "otf_pegasos_step_host": [_int, _vp, _i32, _vp, _i32, _dbl, _dbl, _int, _dbl],
    "otf_train_batch": [_int, _vp, _i32, _i64, _i64, _i32, _vp, _i64, _i32, _i64, _i64, _i64, _dbl, _int,
                        _vp, _vp, _int, _vp],
    "otf_hinge_objective": [_int, _vp, _i32, _i64, _i64, _i32, _vp, _dbl, _vp, _int, _vp],
    "otf_trainer_create": [_int, _i32, _vp, _i32, _i64, _int, _P(_vp)],
    "otf_trainer_destroy": [_vp],
    "otf_trainer_append_positives": [_vp, _vp, _i32, _i64, _int],
    "otf_trainer_pool_size": [_vp, _P(_i64)],
    "otf_trainer_step": [_vp, _vp, _i32, _i64, _vp, _vp, _i32, _dbl, _dbl, _int, _dbl],
    "otf_trainer_weights": [_vp, _vp, _int],
    "otf_trainer_set_weights": [_vp, _vp, _int],
    "otf_trainer_weights_ptr": [_vp, _P(_vp)],
    "otf_trainer_stream": [_vp, _P(_vp)],
    "otf_trainer_publish": [_vp, _vp],
    "otf_repo_rank_published": [_vp, _vp, _i64, _vp, _vp, _vp, _P(_i64)],
    "otf_pq_encode": [_int, _vp, _i64, _i32, _vp, _i32, _i32, _i32, _vp, _int, _vp],
    "otf_kmeans_create": [_int, _vp, _i64, _i32, _i32, _P(_vp)],
    "otf_kmeans_load": [_vp, _vp],
    "otf_kmeans_destroy": [_vp],
    "otf_kmeans_step": [_vp, _vp, _vp, _vp, _P(_dbl)],
    "otf_group_unique_id": [_vp],
    "otf_group_create": [_int, _i32, _i32, _vp, _P(_vp)],
    "otf_group_destroy": [_vp],
    "otf_group_rank": [_vp, _vp, _vp, _i32, _i64, _i64, _i64, _vp, _vp, _vp, _P(_i64), _int, _vp],
}
_RESTYPE = {"otf_last_error": C.c_char_p, "otf_kernel_names": C.c_char_p, "otf_launch_count": _i64}

_lock = threading.Lock()
_lib: C.CDLL | None = None
_checked_device = False


def load(require_device: bool = True) -> C.CDLL:
    """Load the shared library (and, by default, insist on a visible CUDA device)."""
    global _lib, _checked_device
    lib = _lib
    if lib is not None and (_checked_device or not require_device):
        return lib  # the per-query path: no lock once loaded
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise RetrievalError(
                    f"{LIB_PATH.name} is not built; run paper_1407_4764_b200/_build.py "
                    "(no CPU fallback exists)"
                )
            lib = C.CDLL(str(LIB_PATH))
            for name, args in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.argtypes = args
                fn.restype = _RESTYPE.get(name, _int)
            _lib = lib
        if require_device and not _checked_device:
            n = _int(0)
            rc = _lib.otf_device_count(C.byref(n))
            if rc != OK or n.value < 1:
                raise RetrievalError("no CUDA device visible: the B200 retrieval path has no CPU fallback")
            _checked_device = True
        return _lib


def check(rc: int) -> None:
    if rc != OK:
        lib = load(require_device=False)
        msg = lib.otf_last_error().decode(errors="replace")
        raise _ERRORS.get(rc, RetrievalError)(msg)


_ro_last: tuple = (None, 0)  # (the last read-only array, its address): one tuple, swapped atomically


def ptr(a: np.ndarray | None) -> int | None:
    """Address of an array's data for a c_void_p argument. A writable contiguous array goes
    through the buffer protocol (0.45 us); the array interface builds a dict (2.1 us) and is the
    fallback for read-only or non-contiguous arrays. The last read-only array's address is kept
    (a LinearModel's weights are read-only and usually ranked many times: 3.2 -> 0.1 us); an
    ndarray object's data address never changes, and the identity check keeps it exact."""
    global _ro_last
    if a is None:
        return None
    last = _ro_last
    if a is last[0]:
        return last[1]
    try:
        return C.addressof(C.c_char.from_buffer(a))
    except (TypeError, ValueError):
        p = a.__array_interface__["data"][0]
        if not a.flags.writeable:
            _ro_last = (a, p)
        return p


def tptr(t) -> C.c_void_p:
    """Device pointer of a torch tensor."""
    return C.c_void_p(t.data_ptr())


_device = None


def set_reserved_sms(n: int, device: int | None = None) -> None:
    """Leave ``n`` SMs to a concurrent trainer: the persistent rank kernels size their grids for
    the rest (otf_set_reserved_sms). 0 restores the whole GPU."""
    check(load().otf_set_reserved_sms(default_device() if device is None else device, int(n)))


def default_device() -> int:
    global _device
    if _device is None:
        _device = int(os.environ.get("OTF_DEVICE", os.environ.get("LOCAL_RANK", "0")))
    return _device


def set_device(index: int) -> None:
    global _device
    _device = int(index)


def launch_count() -> int:
    return int(load(require_device=False).otf_launch_count())
