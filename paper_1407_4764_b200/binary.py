"""Binary sketches: GPU binarize / unpack / Hamming (reference binary.py:27-128).

``TightFrame`` / ``BinaryCodec`` are containers (the frame's QR construction,
make_tight_frame binary.py:46-66, is offline and out of scope — pass the reference's frame or
any (output_bits, input_dim) float64 matrix). ``binarize`` is the ★-adjacent step that maps
streamed positives into bit space for binary repositories (ranker.py:242-252).
"""

from __future__ import annotations

import dataclasses

import numpy as np

from . import _lib
from .errors import ConfigError


@dataclasses.dataclass(frozen=True)
class TightFrame:
    """Frozen (n, m) projection with orthonormal columns (binary.py:27-43)."""

    matrix: np.ndarray
    seed: int = 0

    @property
    def input_dim(self) -> int:
        return self.matrix.shape[1]

    @property
    def output_bits(self) -> int:
        return self.matrix.shape[0]

    @property
    def code_bytes(self) -> int:
        return (self.output_bits + 7) // 8


@dataclasses.dataclass(frozen=True)
class BinaryCodec:
    """A frame plus the centering vector it thresholds around (binary.py:70-83)."""

    frame: TightFrame
    centering: np.ndarray

    def __post_init__(self):
        center = np.ascontiguousarray(self.centering, dtype=np.float32)
        if center.shape != (self.frame.input_dim,):
            raise ConfigError(
                f"centering shape {center.shape} does not match frame input dim {self.frame.input_dim}"
            )
        center.setflags(write=False)
        object.__setattr__(self, "centering", center)


def binarize(codec, vectors, chunk_rows: int = 1 << 14) -> np.ndarray:
    """binary.py:86-107 — packed LSB-first codes of ((x - mu) U^T > 0), float64 projection."""
    del chunk_rows
    frame = np.ascontiguousarray(codec.frame.matrix, dtype=np.float64)
    n_bits, m = frame.shape
    arr = np.asarray(vectors, dtype=np.float64)
    single = arr.ndim == 1
    if single:
        arr = arr[np.newaxis, :]
    arr = np.ascontiguousarray(arr)
    if arr.shape[1] != m:
        raise ConfigError(f"vector dim {arr.shape[1]} does not match frame input dim {m}")
    mu = np.ascontiguousarray(codec.centering, dtype=np.float32)
    out = np.empty((arr.shape[0], (n_bits + 7) // 8), dtype=np.uint8)
    lib = _lib.load()
    _lib.check(lib.otf_binarize(_lib.default_device(), _lib.ptr(frame), _lib.ptr(mu), m, n_bits,
                                _lib.ptr(arr), arr.shape[0], _lib.ptr(out), _lib.MEM_HOST, None))
    return out[0] if single else out


def unpack_bits(codes, output_bits: int) -> np.ndarray:
    """binary.py:110-120 — (rows, output_bits) float32 {0, 1}, LSB-first, padding dropped."""
    arr = np.asarray(codes, dtype=np.uint8)
    single = arr.ndim == 1
    if single:
        arr = arr[np.newaxis, :]
    arr = np.ascontiguousarray(arr)
    expected = (output_bits + 7) // 8
    if arr.shape[1] != expected:
        raise ConfigError(f"code width {arr.shape[1]} does not match {expected} bytes for {output_bits} bits")
    out = np.empty((arr.shape[0], output_bits), dtype=np.float32)
    lib = _lib.load()
    _lib.check(lib.otf_unpack_bits(_lib.default_device(), _lib.ptr(arr), arr.shape[0], output_bits,
                                   _lib.ptr(out), _lib.MEM_HOST, None))
    return out[0] if single else out


def hamming_distance(a, b) -> np.ndarray:
    """binary.py:123-128 — row-wise Hamming distance between equal-width packed codes."""
    xa = np.ascontiguousarray(np.atleast_2d(np.asarray(a, dtype=np.uint8)))
    xb = np.ascontiguousarray(np.atleast_2d(np.asarray(b, dtype=np.uint8)))
    if xa.shape != xb.shape:
        raise ConfigError(f"code shapes {xa.shape} and {xb.shape} differ")
    out = np.empty(xa.shape[0], dtype=np.int64)
    lib = _lib.load()
    _lib.check(lib.otf_hamming(_lib.default_device(), _lib.ptr(xa), _lib.ptr(xb), xa.shape[0], xa.shape[1],
                               _lib.ptr(out), _lib.MEM_HOST, None))
    return out if np.ndim(a) > 1 else out[0]
