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
