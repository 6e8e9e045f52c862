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
import dataclasses

import numpy as np

from . import _lib
from .errors import ConfigError, InsufficientDataError

DEFAULT_NUM_CENTROIDS = 256
DEFAULT_ITERATIONS = 25


@dataclasses.dataclass(frozen=True)
class PQConfig:
    """pq.py:28-48 — codebook learning knobs."""

    subdim: int
    num_centroids: int = DEFAULT_NUM_CENTROIDS
    iterations: int = DEFAULT_ITERATIONS
    seed: int = 0

    def validate(self) -> None:
        if self.subdim <= 0:
            raise ConfigError(f"subdim must be positive, got {self.subdim}")
        if not 1 <= self.num_centroids <= 256:
            raise ConfigError(f"num_centroids must be in [1, 256], got {self.num_centroids}")
        if self.iterations < 0:
            raise ConfigError(f"iterations must be >= 0, got {self.iterations}")


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
        self.objective_history: list[list[float]] = []

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


class _KMeansBlock:
    """One block's float64 training sub-vectors on the device (otf_kmeans_*)."""

    def __init__(self, data: np.ndarray, k: int):
        self.data = np.ascontiguousarray(data, dtype=np.float64)
        self.k = int(k)
        h = C.c_void_p()
        _lib.check(_lib.load().otf_kmeans_create(_lib.default_device(), _lib.ptr(self.data), self.data.shape[0],
                                                 self.data.shape[1], self.k, C.byref(h)))
        self._h = h

    def load(self, data: np.ndarray) -> None:
        """Swap in another block of the same shape (one handle serves every block)."""
        self.data = np.ascontiguousarray(data, dtype=np.float64)
        _lib.check(_lib.load().otf_kmeans_load(self._h, _lib.ptr(self.data)))

    def step(self, centroids: np.ndarray):
        """(assign, counts, objective, plain-updated centroids) for the given centroids."""
        c = np.ascontiguousarray(centroids, dtype=np.float64).copy()
        assign = np.empty(self.data.shape[0], dtype=np.int32)
        counts = np.empty(self.k, dtype=np.int64)
        obj = C.c_double()
        _lib.check(_lib.load().otf_kmeans_step(self._h, _lib.ptr(c), _lib.ptr(assign), _lib.ptr(counts),
                                               C.byref(obj)))
        return assign.astype(np.int64), counts, float(obj.value), c

    def close(self) -> None:
        if getattr(self, "_h", None) is not None and self._h.value and _lib._lib is not None:
            _lib._lib.otf_kmeans_destroy(self._h)
        self._h = None

    def __del__(self):
        self.close()


def _sorted_unique_rows(x: np.ndarray) -> np.ndarray:
    """np.unique(x, axis=0): rows in lexicographic float order, exact duplicates removed.

    numpy sorts the rows as structured records (~0.1 s at 50k rows). Here: one argsort of the
    first column, then only the groups that tie on it are ordered by the remaining columns.
    With NaN or -0.0 anywhere (where numpy's representative among rows that compare equal but
    differ in bits depends on its unstable sort) numpy's own path runs instead."""
    if x.shape[0] <= 1 or x.shape[1] == 0 or np.isnan(x).any() or (np.signbit(x) & (x == 0)).any():
        return np.unique(x, axis=0)
    s = x[np.argsort(x[:, 0], kind="stable")]
    tie = s[1:, 0] == s[:-1, 0]
    if tie.any():
        starts = np.flatnonzero(np.concatenate([[True], ~tie]))
        ends = np.append(starts[1:], len(s))
        for a, b in zip(starts[ends - starts > 1], ends[ends - starts > 1]):
            g = s[a:b]
            s[a:b] = g[np.lexsort(g.T[::-1])]
        keep = np.ones(len(s), dtype=bool)
        keep[1:] = np.any(s[1:] != s[:-1], axis=1)
        s = s[keep]
    return s


def _lloyd(block, k: int, iterations: int, rng: np.random.Generator, init=None, _km=None):
    """pq.py:116-171 — plain Lloyd iterations on one sub-block, float64; the assignment, the
    objective and the means run on the GPU (csrc/otf_kmeans.cu), the initial pick and the rare
    empty-cluster re-seed run here exactly as the reference writes them."""
    data = np.asarray(block, dtype=np.float64)
    if init is None:
        unique_rows = _sorted_unique_rows(data)
        if unique_rows.shape[0] < k:
            raise InsufficientDataError(f"need at least {k} distinct sub-vectors, found {unique_rows.shape[0]}")
        pick = rng.choice(unique_rows.shape[0], size=k, replace=False)
        centroids = unique_rows[pick].copy()
    else:
        centroids = np.asarray(init, dtype=np.float64).copy()
        if centroids.shape != (k, data.shape[1]):
            raise ConfigError(f"init shape {centroids.shape} does not match (k, subdim)")
    history: list[float] = []
    if iterations == 0:
        return centroids, history
    if _km is not None:  # learn_pq_codebook's shared handle (device buffers reused across blocks)
        km = _km
        km.load(data)
    else:
        km = _KMeansBlock(data, k)
    try:
        prev_assign = None
        plain_update = True
        for _ in range(iterations):
            assign, counts, obj, means = km.step(centroids)
            history.append(obj)
            if prev_assign is not None and plain_update and np.array_equal(assign, prev_assign):
                break
            prev_assign = assign
            empties = np.flatnonzero(counts == 0)
            plain_update = empties.size == 0
            centroids = means
            for j in empties:
                largest = int(np.argmax(counts))
                members = np.flatnonzero(assign == largest)
                gaps = np.sum((data[members] - centroids[largest]) ** 2, axis=1)
                stolen = members[int(np.argmax(gaps))]
                centroids[j] = data[stolen]
                assign[stolen] = j
                counts[largest] -= 1
                counts[j] += 1
    finally:
        if _km is None:
            km.close()
    return centroids, history


def learn_pq_codebook(train, cfg: PQConfig) -> PQCodebook:
    """pq.py:174-203 — one k-means codebook per sub-block, blocks in order on one seeded rng."""
    cfg.validate()
    data = train.data if hasattr(train, "data") and not isinstance(train, np.ndarray) else np.asarray(
        train, dtype=np.float32)
    data = np.asarray(data, dtype=np.float32)
    if data.ndim != 2 or data.shape[0] == 0:
        raise ConfigError("training data must be a non-empty 2-D array")
    dim = data.shape[1]
    if dim % cfg.subdim != 0:
        raise ConfigError(f"dim {dim} is not divisible by subdim {cfg.subdim}")
    if data.shape[0] < cfg.num_centroids:
        raise InsufficientDataError(f"{data.shape[0]} training vectors for {cfg.num_centroids} centroids")
    rng = np.random.default_rng(cfg.seed)
    blocks = dim // cfg.subdim
    centroids = np.empty((blocks, cfg.num_centroids, cfg.subdim), dtype=np.float32)
    histories: list[list[float]] = []
    km = _KMeansBlock(data[:, :cfg.subdim], cfg.num_centroids) if cfg.iterations > 0 else None
    try:
        for m in range(blocks):
            sub = data[:, m * cfg.subdim:(m + 1) * cfg.subdim]
            cents, history = _lloyd(sub, cfg.num_centroids, cfg.iterations, rng, _km=km)
            centroids[m] = cents.astype(np.float32)
            histories.append(history)
    finally:
        if km is not None:
            km.close()
    centering = data.astype(np.float64).mean(axis=0).astype(np.float32)
    book = PQCodebook(centroids, centering)
    book.objective_history = histories
    return book
