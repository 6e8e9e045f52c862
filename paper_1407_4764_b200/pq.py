"""Product-quantized scoring on the GPU (reference pq.py:51-97, :248-276).

``build_score_lut`` and ``score_codes`` keep the reference's signatures and return the
reference's float64 values bit-for-bit: the CUDA kernels (csrc/otf_pq.cu) replay numpy's
einsum and pairwise-sum orders. ``pq_encode`` (pq.py:206-230, the ingest path of a PQ
repository) runs on the GPU too. Codebook learning and the OTFQ/OTFC formats
are offline and out of scope; ``PQCodebook`` here is the container only, and any
object with ``centroids`` / ``num_blocks`` / ``num_centroids`` / ``subdim`` works (e.g. the
reference's own PQCodebook).
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .errors import ConfigError


class PQCodebook:
    """(num_blocks, num_centroids, subdim) float32 centroids + centering (pq.py:51-97)."""

    def __init__(self, centroids, centering=None):
        cents = np.ascontiguousarray(centroids, dtype=np.float32)
        if cents.ndim != 3:
            raise ConfigError(f"centroids must be (blocks, centroids, subdim), got {cents.shape}")
        dim = cents.shape[0] * cents.shape[2]
        center = np.zeros(dim, np.float32) if centering is None else np.ascontiguousarray(centering, dtype=np.float32)
        if center.shape != (dim,):
            raise ConfigError(f"centering length {center.shape} does not match dim {dim}")
        cents.setflags(write=False)
        center.setflags(write=False)
        self._centroids = cents
        self._centering = center

    @property
    def centroids(self) -> np.ndarray:
        return self._centroids

    @property
    def centering(self) -> np.ndarray:
        return self._centering

    @property
    def num_blocks(self) -> int:
        return self._centroids.shape[0]

    @property
    def num_centroids(self) -> int:
        return self._centroids.shape[1]

    @property
    def subdim(self) -> int:
        return self._centroids.shape[2]

    @property
    def dim(self) -> int:
        return self.num_blocks * self.subdim


def _centroids(codebook) -> np.ndarray:
    return np.ascontiguousarray(codebook.centroids, dtype=np.float32)


def build_score_lut(weights, codebook) -> np.ndarray:
    """pq.py:248-259 — (num_blocks, num_centroids) float64 LUT, numpy-einsum bit-exact."""
    w = np.ascontiguousarray(weights, dtype=np.float64)
    cents = _centroids(codebook)
    m, k, q = cents.shape
    if w.shape != (m * q,):
        raise ConfigError(f"weights shape {w.shape} does not match codebook dim {m * q}")
    lib = _lib.load()
    out = np.empty((m, k), dtype=np.float64)
    _lib.check(lib.otf_pq_build_lut(_lib.default_device(), _lib.ptr(cents), m, k, q, _lib.ptr(w),
                                    _lib.ptr(out), _lib.MEM_HOST, None))
    return out


def score_codes(lut, codes, chunk_rows: int = 1 << 18) -> np.ndarray:
    """pq.py:262-276 — float64 LUT-sum scores, numpy pairwise-sum bit-exact.

    ``chunk_rows`` is accepted for signature parity; the GPU scans all rows in one pass.
    """
    del chunk_rows
    table = np.ascontiguousarray(lut, dtype=np.float64)
    arr = np.asarray(codes, dtype=np.uint8)
    single = arr.ndim == 1
    if single:
        arr = arr[np.newaxis, :]
    arr = np.ascontiguousarray(arr)
    m, k = table.shape
    if arr.shape[1] != m:
        raise ConfigError(f"code width {arr.shape[1]} does not match LUT with {m} blocks")
    lib = _lib.load()
    out = np.empty(arr.shape[0], dtype=np.float64)
    _lib.check(lib.otf_pq_score_codes(_lib.default_device(), _lib.ptr(table), m, k, _lib.ptr(arr),
                                      arr.shape[0], _lib.ptr(out), _lib.MEM_HOST, None))
    return out[0] if single else out


def pq_encode(codebook, vectors, chunk_rows: int = 1 << 18) -> np.ndarray:
    """pq.py:206-230 — (n, num_blocks) uint8 codes, nearest centroid per block in float64.

    A single (dim,) vector gives a (num_blocks,) code. ``chunk_rows`` is accepted for signature
    parity (the GPU encodes all rows in one launch). The distance |c|^2 - 2 x.c is the
    reference's; only its Q-term dot may round differently from OpenBLAS's, so a code can differ
    only where two centroids are equidistant to rounding level.
    """
    del chunk_rows
    cents = _centroids(codebook)
    m, k, q = cents.shape
    arr = np.asarray(vectors, dtype=np.float32)
    single = arr.ndim == 1
    if single:
        arr = arr[np.newaxis, :]
    arr = np.ascontiguousarray(arr)
    if arr.shape[1] != m * q:
        raise ConfigError(f"vector dim {arr.shape[1]} does not match codebook dim {m * q}")
    out = np.empty((arr.shape[0], m), dtype=np.uint8)
    if arr.shape[0]:
        _lib.check(_lib.load().otf_pq_encode(_lib.default_device(), _lib.ptr(arr), arr.shape[0], arr.shape[1],
                                             _lib.ptr(cents), m, k, q, _lib.ptr(out), _lib.MEM_HOST, None))
    return out[0] if single else out
