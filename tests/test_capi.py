"""CPU checks of the C ABI boundary: the library builds for sm_100a, loads, exports every symbol
declared in include/otf_b200.h, and the product path refuses to run without a GPU (no fallback)."""

import ctypes
import re
import subprocess
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "otf_b200.h"


def declared_functions():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[\w\s\*]+?\b(otf_\w+)\s*\(", text, flags=re.M)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for required in ["otf_repo_create_dense", "otf_repo_create_pq", "otf_repo_create_binary", "otf_repo_rank",
                     "otf_repo_score", "otf_top_k", "otf_pegasos_update", "otf_trainer_step",
                     "otf_pq_build_lut", "otf_pq_score_codes", "otf_score_binary", "otf_binarize"]:
        assert required in names


def test_library_exports_every_declared_symbol(built_lib):
    lib = ctypes.CDLL(str(built_lib))
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert missing == []


def test_library_is_sm100a_code(built_lib):
    out = subprocess.run(["cuobjdump", "--list-elf", str(built_lib)], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_python_bindings_match_header(built_lib):
    from paper_1407_4764_b200 import _lib

    assert set(_lib.SIGNATURES) == set(declared_functions())


def test_no_cpu_fallback_without_device(built_lib):
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    import paper_1407_4764_b200 as otf

    with pytest.raises(otf.RetrievalError):
        otf.score_dense(np.zeros(4), np.ones((3, 4), np.float32))
    with pytest.raises(otf.RetrievalError):
        otf.top_k(np.ones(5), 2)


def test_status_codes_map_to_the_reference_exceptions(built_lib):
    """include/otf_b200.h status codes -> errors.py classes (incl. the file loaders' FormatError,
    DegenerateInputError and OSError)."""
    from paper_1407_4764_b200 import _lib, errors

    text = HEADER.read_text()
    codes = {name: int(v) for name, v in re.findall(r"#define (OTF_ERR_\w+) (\d+)", text)}
    want = {"OTF_ERR_CONFIG": errors.ConfigError, "OTF_ERR_NOT_READY": errors.NotReadyError,
            "OTF_ERR_INSUFFICIENT": errors.InsufficientDataError, "OTF_ERR_CORRUPTION": errors.CorruptionError,
            "OTF_ERR_EMPTY": errors.EmptyStoreError, "OTF_ERR_CUDA": errors.RetrievalError,
            "OTF_ERR_NCCL": errors.RetrievalError, "OTF_ERR_FORMAT": errors.FormatError,
            "OTF_ERR_DEGENERATE": errors.DegenerateInputError, "OTF_ERR_IO": OSError}
    assert set(codes) == set(want)
    for name, cls in want.items():
        assert _lib._ERRORS[codes[name]] is cls


def test_array_pointer_helper():
    """_lib.ptr: the buffer-protocol fast path and the array-interface fallback give the same
    address (writable, read-only, strided and empty arrays)."""
    from paper_1407_4764_b200 import _lib

    a = np.arange(10.0)
    ro = np.arange(6.0)
    ro.setflags(write=False)
    for x in (a, a[2:], a[::2], ro, np.empty(0), np.zeros((3, 4), np.float32)):
        assert _lib.ptr(x) == x.__array_interface__["data"][0]
    assert _lib.ptr(None) is None


def test_loader_header_peek(tmp_path):
    """Repository._file_header reads the (count, width) fields the ids check needs; anything
    that is not a complete header of the expected magic is left to the C loader's errors."""
    import struct

    from paper_1407_4764_b200 import Repository

    p = tmp_path / "c.otfc"
    p.write_bytes(b"OTFC" + struct.pack("<I", 1) + struct.pack("<Q", 7) + struct.pack("<I", 16) + bytes(7 * 16))
    assert Repository._file_header(p, b"OTFC") == (7, 16)
    assert Repository._file_header(p, b"OTFH") == (None, None)
    p.write_bytes(b"OTFC")
    assert Repository._file_header(p, b"OTFC") == (None, None)
    with pytest.raises(FileNotFoundError):
        Repository._file_header(tmp_path / "missing.otfc", b"OTFC")
