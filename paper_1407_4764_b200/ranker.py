"""GPU scoring and exact top-k ranking — drop-in for the reference's ranker.py:1-281.

Same names, signatures, return types and error types as the reference module:
``score_dense`` / ``score_pq`` / ``score_binary`` / ``top_k`` / ``RankedList`` /
``RankerConfig`` / ``Repository``. The difference is where the data lives: a ``Repository``
copies its payload (dense float32 rows, PQ byte codes or packed bits) into HBM once, and every
``score`` / ``rank`` is a scan by the sm_100a kernels behind the C ABI (include/otf_b200.h).
There is no CPU path.
"""

from __future__ import annotations

import ctypes as C
import dataclasses
import struct
from pathlib import Path
from typing import Iterator

import numpy as np

from . import _lib
from .binary import binarize, unpack_bits
from .errors import ConfigError, CorruptionError
from .model import LinearModel, as_weights, model_version

DEFAULT_LIST_SIZE = 100
DEFAULT_RANK_INTERVAL = 0.18


@dataclasses.dataclass(frozen=True)
class RankerConfig:
    """ranker.py:28-39 — list size and re-rank cadence of live sessions."""

    k: int = DEFAULT_LIST_SIZE
    interval: float = DEFAULT_RANK_INTERVAL

    def validate(self) -> None:
        if self.k < 1:
            raise ConfigError(f"k must be >= 1, got {self.k}")
        if self.interval <= 0:
            raise ConfigError(f"interval must be positive, got {self.interval}")


@dataclasses.dataclass(frozen=True)
class RankedList:
    """ranker.py:42-56 — ids (int64), scores (float64), provenance, optional names."""

    ids: np.ndarray
    scores: np.ndarray
    model_version: int
    produced_at: float
    names: tuple | None = None

    def __len__(self) -> int:
        return len(self.ids)

    def entries(self) -> Iterator[tuple[int, float]]:
        return zip((int(i) for i in self.ids), (float(s) for s in self.scores))

    @classmethod
    def _make(cls, ids, scores, model_version, produced_at, names=None) -> "RankedList":
        """The per-query constructor: the same fields without the frozen dataclass's five
        object.__setattr__ calls (1.8 -> 1.0 us)."""
        obj = object.__new__(cls)
        d = obj.__dict__
        d["ids"] = ids
        d["scores"] = scores
        d["model_version"] = model_version
        d["produced_at"] = produced_at
        d["names"] = names
        return obj


def _f32_rows(store) -> np.ndarray:
    data = store.data if hasattr(store, "data") else store
    return np.ascontiguousarray(np.asarray(data, dtype=np.float32))


def score_dense(model, store) -> np.ndarray:
    """ranker.py:63-69 — float32 scores <x, float32(w)> (float64 accumulation on the GPU)."""
    x = _f32_rows(store)
    w = as_weights(model)
    if x.ndim != 2 or x.shape[1] != w.shape[0]:
        raise ConfigError(f"store dim {x.shape[1] if x.ndim == 2 else x.shape} does not match model dim {w.shape[0]}")
    out = np.empty(x.shape[0], dtype=np.float32)
    lib = _lib.load()
    _lib.check(lib.otf_score_dense(_lib.default_device(), _lib.ptr(x), x.shape[0], x.shape[1], _lib.ptr(w),
                                   _lib.ptr(out), _lib.MEM_HOST, None))
    return out


def score_pq(model, codebook, codes) -> np.ndarray:
    """ranker.py:72-75 — LUT scoring of quantized vectors (float64, bit-exact)."""
    from .pq import build_score_lut, score_codes

    return score_codes(build_score_lut(as_weights(model), codebook), codes)


def score_binary(model, codes, output_bits: int, chunk_rows: int = 1 << 14) -> np.ndarray:
    """ranker.py:78-94 — sum of float32(w_j) over set bits j (LSB-first), float32 out."""
    del chunk_rows
    w = as_weights(model)
    if w.shape[0] != output_bits:
        raise ConfigError(f"model dim {w.shape[0]} does not match {output_bits} code bits")
    arr = np.ascontiguousarray(np.asarray(codes, dtype=np.uint8))
    if arr.ndim != 2 or arr.shape[1] != (output_bits + 7) // 8:
        raise ConfigError(f"codes shape {arr.shape} does not match {output_bits} bits")
    out = np.empty(arr.shape[0], dtype=np.float32)
    lib = _lib.load()
    _lib.check(lib.otf_score_binary(_lib.default_device(), _lib.ptr(arr), arr.shape[0], output_bits, _lib.ptr(w),
                                    _lib.ptr(out), _lib.MEM_HOST, None))
    return out


def _empty_list(model_version_: int, produced_at: float, names) -> RankedList:
    return RankedList(np.empty(0, dtype=np.int64), np.empty(0, dtype=np.float64), model_version_, produced_at,
                      tuple() if names is not None else None)


def top_k(scores, k: int, ids=None, names=None, model_version: int = 0, produced_at: float = 0.0) -> RankedList:
    """ranker.py:97-143 — the first k of a full sort by (-score, id), on the GPU."""
    s = np.asarray(scores)
    if s.dtype != np.float32:
        s = s.astype(np.float64)
    s = np.ascontiguousarray(s)
    n = s.shape[0]
    id_arr = None
    if ids is not None:
        id_arr = np.ascontiguousarray(np.asarray(ids, dtype=np.int64))
        if id_arr.shape != (n,):
            raise ConfigError(f"ids shape {id_arr.shape} does not match {n} scores")
    k_eff = max(0, min(int(k), n))
    if k_eff == 0:
        return _empty_list(model_version, produced_at, names)
    out_ids = np.empty(k_eff, dtype=np.int64)
    out_sc = np.empty(k_eff, dtype=np.float64)
    out_rows = np.empty(k_eff, dtype=np.int64)
    got = C.c_int64(0)
    lib = _lib.load()
    _lib.check(lib.otf_top_k(_lib.default_device(), _lib.ptr(s), _lib.F32 if s.dtype == np.float32 else _lib.F64,
                             n, _lib.ptr(id_arr), k_eff, _lib.ptr(out_ids), _lib.ptr(out_sc), _lib.ptr(out_rows),
                             C.byref(got), _lib.MEM_HOST, None))
    out_names = tuple(names[int(r)] for r in out_rows) if names is not None else None
    return RankedList(out_ids, out_sc, model_version, produced_at, out_names)


class Repository:
    """ranker.py:146-281 — a GPU-resident repository in one of three representations.

    The payload is copied into HBM once at construction (or adopted in place from a device
    pointer, see ``from_device``); ``score`` and ``rank`` stream it through the kernels.
    """

    def __init__(self, kind: str, handle: C.c_void_p, model_dim: int, ids, names, codebook=None, codec=None,
                 output_bits=None):
        self.kind = kind
        self._handle = handle
        self._model_dim = int(model_dim)
        # ids: an int64 array, or an int n for the implicit 0..n-1 (built on first access: a file
        # loader's 100M-row repository does not pay an 800 MB host array it may never read)
        self._ids = ids if isinstance(ids, int) else np.asarray(ids, dtype=np.int64)
        self.names = list(names) if names is not None else None
        self._codebook = codebook
        self._codec = codec
        self._output_bits = output_bits

    # -- constructors (ranker.py:176-209) ----------------------------------------------------
    @classmethod
    def dense(cls, store, device: int | None = None) -> "Repository":
        x = _f32_rows(store)
        if x.ndim != 2:
            raise ConfigError(f"feature data must be 2-D, got shape {x.shape}")
        n, d = x.shape
        ids = getattr(store, "ids", None)
        ids = np.arange(n, dtype=np.int64) if ids is None else np.ascontiguousarray(ids, dtype=np.int64)
        names = getattr(store, "names", None)
        dev = _lib.default_device() if device is None else device
        h = C.c_void_p()
        lib = _lib.load()
        _lib.check(lib.otf_repo_create_dense(dev, _lib.ptr(x), n, d, _lib.ptr(ids), 0, _lib.MEM_HOST, 0,
                                             C.byref(h)))
        return cls("dense", h, d, ids, names)

    @classmethod
    def quantized(cls, codebook, codes, ids=None, names=None, device: int | None = None) -> "Repository":
        codes = np.ascontiguousarray(np.asarray(codes, dtype=np.uint8))
        if codes.ndim != 2 or codes.shape[1] != codebook.num_blocks:
            raise ConfigError(f"codes shape {codes.shape} does not match {codebook.num_blocks} blocks")
        ids = np.arange(codes.shape[0], dtype=np.int64) if ids is None else np.ascontiguousarray(ids, dtype=np.int64)
        cents = np.ascontiguousarray(codebook.centroids, dtype=np.float32)
        m, k, q = cents.shape
        dev = _lib.default_device() if device is None else device
        h = C.c_void_p()
        lib = _lib.load()
        _lib.check(lib.otf_repo_create_pq(dev, _lib.ptr(codes), codes.shape[0], _lib.ptr(cents), m, k, q,
                                          _lib.ptr(ids), 0, _lib.MEM_HOST, 0, C.byref(h)))
        return cls("pq", h, m * q, ids, names, codebook=codebook)

    @classmethod
    def binary(cls, codec, codes, ids=None, names=None, device: int | None = None) -> "Repository":
        codes = np.ascontiguousarray(np.asarray(codes, dtype=np.uint8))
        bits = codec.frame.output_bits
        if codes.ndim != 2 or codes.shape[1] != codec.frame.code_bytes:
            raise ConfigError(f"codes shape {codes.shape} does not match {bits} bits")
        ids = np.arange(codes.shape[0], dtype=np.int64) if ids is None else np.ascontiguousarray(ids, dtype=np.int64)
        dev = _lib.default_device() if device is None else device
        h = C.c_void_p()
        lib = _lib.load()
        _lib.check(lib.otf_repo_create_binary(dev, _lib.ptr(codes), codes.shape[0], bits, _lib.ptr(ids), 0,
                                              _lib.MEM_HOST, 0, C.byref(h)))
        return cls("binary", h, bits, ids, names, codec=codec, output_bits=bits)

    @property
    def ids(self) -> np.ndarray:
        if isinstance(self._ids, int):
            self._ids = np.arange(self._ids, dtype=np.int64)
        return self._ids

    # -- repository files straight into HBM (§8 f3; otf_ingest.cu) ------------------------------
    @staticmethod
    def _file_header(path, magic: bytes):
        """(u64, u32) header fields of an OTFC / OTFH file, for the ids-length check (the C loader
        re-validates everything, formats.py:40-84)."""
        with open(path, "rb") as fh:  # FileNotFoundError / IsADirectoryError as the reference's open()
            head = fh.read(20)
        if len(head) < 20 or head[:4] != magic:
            return None, None
        return struct.unpack("<Q", head[8:16])[0], struct.unpack("<I", head[16:20])[0]

    @classmethod
    def load_features(cls, path, normalize: bool = True, device: int | None = None) -> "Repository":
        """Repository.dense(load_features(path, normalize)) without a host copy of the rows:
        store.py:139-163 (OTFR; rows L2-normalised on the device exactly as normalize_rows,
        store.py:32-53; the ``.names`` sidecar as the reference), ranker.py:176-178."""
        path = Path(path)
        open(path, "rb").close()  # the reference's open() errors
        dev = _lib.default_device() if device is None else device
        h = C.c_void_p()
        _lib.check(_lib.load().otf_repo_load_dense(dev, str(path).encode(), int(bool(normalize)), C.byref(h)))
        kind, count, dim, nbytes, d = C.c_int32(), C.c_int64(), C.c_int32(), C.c_int64(), C.c_int32()
        _lib.check(_lib.load().otf_repo_info(h, C.byref(kind), C.byref(count), C.byref(dim), C.byref(nbytes),
                                             C.byref(d)))
        names = None
        names_path = path.with_suffix(path.suffix + ".names")
        if names_path.exists():
            names = names_path.read_text(encoding="utf-8").splitlines()
            if len(names) != count.value:
                _lib.load().otf_repo_destroy(h)
                raise CorruptionError(f"{names_path}: {len(names)} names for {count.value} rows")
        return cls("dense", h, dim.value, count.value, names)

    @classmethod
    def load_quantized(cls, codebook, path, ids=None, names=None, device: int | None = None) -> "Repository":
        """Repository.quantized(codebook, load_pq_codes(path, codebook.num_centroids), ids, names)
        without a host copy of the codes: pq.py:318-330 (OTFC), ranker.py:180-192."""
        count, _ = cls._file_header(path, b"OTFC")
        cents = np.ascontiguousarray(codebook.centroids, dtype=np.float32)
        m, k, q = cents.shape
        id_arr = None
        if ids is not None:
            id_arr = np.ascontiguousarray(ids, dtype=np.int64)
            if count is not None and id_arr.shape != (count,):
                raise ConfigError(f"ids shape {id_arr.shape} does not match {count} codes")
        dev = _lib.default_device() if device is None else device
        h = C.c_void_p()
        _lib.check(_lib.load().otf_repo_load_pq(dev, str(path).encode(), _lib.ptr(cents), m, k, q, _lib.ptr(id_arr),
                                                C.byref(h)))
        ids_host = id_arr if id_arr is not None else cls._handle_count(h)
        return cls("pq", h, m * q, ids_host, names, codebook=codebook)

    @classmethod
    def load_binary(cls, codec, path, ids=None, names=None, device: int | None = None) -> "Repository":
        """Repository.binary(codec, load_binary_codes(path)[0], ids, names) without a host copy of
        the codes: binary.py:176-187 (OTFH, padding bits checked on the device), ranker.py:194-209."""
        count, _ = cls._file_header(path, b"OTFH")
        bits = codec.frame.output_bits
        id_arr = None
        if ids is not None:
            id_arr = np.ascontiguousarray(ids, dtype=np.int64)
            if count is not None and id_arr.shape != (count,):
                raise ConfigError(f"ids shape {id_arr.shape} does not match {count} codes")
        dev = _lib.default_device() if device is None else device
        h = C.c_void_p()
        got = C.c_int32()
        _lib.check(_lib.load().otf_repo_load_binary(dev, str(path).encode(), codec.frame.code_bytes, _lib.ptr(id_arr),
                                                    C.byref(h), C.byref(got)))
        ids_host = id_arr if id_arr is not None else cls._handle_count(h)
        return cls("binary", h, bits, ids_host, names, codec=codec, output_bits=bits)

    @staticmethod
    def _handle_count(h) -> int:
        kind, count, dim, nbytes, d = C.c_int32(), C.c_int64(), C.c_int32(), C.c_int64(), C.c_int32()
        _lib.check(_lib.load().otf_repo_info(h, C.byref(kind), C.byref(count), C.byref(dim), C.byref(nbytes),
                                             C.byref(d)))
        return count.value

    @classmethod
    def from_device(cls, kind: str, data_ptr: int, count: int, dim: int, *, ids=None, id_base: int = 0,
                    names=None, codebook=None, codec=None, device: int | None = None,
                    borrow: bool = True) -> "Repository":
        """Adopt a payload already in HBM (e.g. a torch CUDA tensor's data_ptr()).

        ``dim`` is the feature dim (dense), num_blocks (pq) or output_bits (binary). With
        ``borrow`` the handle reads the caller's buffer in place (the caller keeps it alive).
        ``ids`` (host int64) default to ``id_base + row`` — the sharded layout of §8(e).
        """
        dev = _lib.default_device() if device is None else device
        id_arr = None if ids is None else np.ascontiguousarray(ids, dtype=np.int64)
        h = C.c_void_p()
        lib = _lib.load()
        p = C.c_void_p(int(data_ptr))
        if kind == "dense":
            _lib.check(lib.otf_repo_create_dense(dev, p, count, dim, _lib.ptr(id_arr), id_base, _lib.MEM_DEVICE,
                                                 int(borrow), C.byref(h)))
            model_dim = dim
        elif kind == "pq":
            cents = np.ascontiguousarray(codebook.centroids, dtype=np.float32)
            m, k, q = cents.shape
            if m != dim:
                raise ConfigError(f"codes width {dim} does not match {m} blocks")
            _lib.check(lib.otf_repo_create_pq(dev, p, count, _lib.ptr(cents), m, k, q, _lib.ptr(id_arr), id_base,
                                              _lib.MEM_DEVICE, int(borrow), C.byref(h)))
            model_dim = m * q
        elif kind == "binary":
            _lib.check(lib.otf_repo_create_binary(dev, p, count, dim, _lib.ptr(id_arr), id_base, _lib.MEM_DEVICE,
                                                  int(borrow), C.byref(h)))
            model_dim = dim
        else:
            raise ConfigError(f"unknown repository kind {kind!r}")
        ids_host = id_arr if id_arr is not None else np.arange(id_base, id_base + count, dtype=np.int64)
        return cls(kind, h, model_dim, ids_host, names, codebook=codebook, codec=codec,
                   output_bits=dim if kind == "binary" else None)

    def __del__(self):
        h = getattr(self, "_handle", None)
        if h is not None and h.value and _lib._lib is not None:
            _lib._lib.otf_repo_destroy(h)
            self._handle = None

    # -- views (ranker.py:213-231) ------------------------------------------------------------
    def _info(self):
        # (count, payload bytes, device) never change for a handle: one C call per repository
        info = self.__dict__.get("_info_cache")
        if info is None:
            kind, count, dim, nbytes, dev = C.c_int32(), C.c_int64(), C.c_int32(), C.c_int64(), C.c_int32()
            _lib.check(_lib.load().otf_repo_info(self._handle, C.byref(kind), C.byref(count), C.byref(dim),
                                                 C.byref(nbytes), C.byref(dev)))
            info = self._info_cache = (count.value, nbytes.value, dev.value)
        return info

    @property
    def handle(self) -> C.c_void_p:
        """The C ABI handle (otf_repo*) for callers that drive the library directly."""
        return self._handle

    @property
    def device(self) -> int:
        return self._info()[2]

    @property
    def count(self) -> int:
        return self._info()[0]

    @property
    def model_dim(self) -> int:
        return self._model_dim

    @property
    def feature_dim(self) -> int:
        if self.kind == "binary":
            return self._codec.frame.input_dim
        return self._model_dim

    def payload_bytes(self) -> int:
        return int(self._info()[1])

    # -- scoring / ranking (ranker.py:233-281) -----------------------------------------------
    def _weights(self, model) -> np.ndarray:
        w = as_weights(model)
        if w.shape != (self._model_dim,):
            if self.kind == "binary":
                raise ConfigError(f"model dim {w.shape[0]} does not match {self._model_dim} code bits")
            raise ConfigError(f"store dim {self._model_dim} does not match model dim {w.shape[0]}")
        return w

    def score(self, model) -> np.ndarray:
        w = self._weights(model)
        n = self.count
        out = np.empty(n, dtype=np.float64 if self.kind == "pq" else np.float32)
        _lib.check(_lib.load().otf_repo_score(self._handle, _lib.ptr(w), _lib.ptr(out), _lib.MEM_HOST, None))
        return out

    def adapt_training_vectors(self, vectors) -> np.ndarray:
        """ranker.py:242-252: identity for dense/PQ; binarize + unpack for binary."""
        arr = np.asarray(vectors, dtype=np.float32)
        if self.kind != "binary":
            return arr
        return unpack_bits(binarize(self._codec, arr), self._output_bits)

    def without_ids(self, excluded) -> "Repository":
        """ranker.py:254-270: a new repository without the excluded ids (rows gathered on device)."""
        drop = np.fromiter((int(i) for i in excluded), dtype=np.int64)
        if drop.size == 0:
            return self
        keep = np.flatnonzero(~np.isin(self.ids, drop)).astype(np.int64)
        h = C.c_void_p()
        _lib.check(_lib.load().otf_repo_subset(self._handle, _lib.ptr(keep), keep.size, C.byref(h)))
        names = [self.names[i] for i in keep] if self.names is not None else None
        return Repository(self.kind, h, self._model_dim, self.ids[keep], names, codebook=self._codebook,
                          codec=self._codec, output_bits=self._output_bits)

    # -- many classifiers at once (C5b; tensor cores, dense repositories) -------------------------
    def _weight_matrix(self, models) -> np.ndarray:
        rows = [as_weights(m) for m in models]
        W = np.ascontiguousarray(np.stack(rows), dtype=np.float64)
        if W.ndim != 2 or W.shape[1] != self._model_dim:
            raise ConfigError(f"store dim {self._model_dim} does not match model dim {W.shape[-1]}")
        return W

    def score_many(self, models) -> np.ndarray:
        """(len(models), count) float32 scores — one score_dense per model (ranker.py:63-69),
        computed together on the tcgen05 tensor cores (TF32 with a 3-product split)."""
        W = self._weight_matrix(models)
        out = np.empty((W.shape[0], self.count), dtype=np.float32)
        _lib.check(_lib.load().otf_repo_score_many(self._handle, _lib.ptr(W), W.shape[0], _lib.ptr(out),
                                                   _lib.MEM_HOST, None))
        return out

    def rank_many(self, models, k: int, produced_at: float = 0.0) -> list[RankedList]:
        """[self.rank(m, k) for m in models], scored together on the tensor cores."""
        W = self._weight_matrix(models)
        k_eff = max(0, min(int(k), self.count))
        ids = np.empty((W.shape[0], k_eff), dtype=np.int64)
        sc = np.empty((W.shape[0], k_eff), dtype=np.float64)
        got = C.c_int64(0)
        if k_eff:
            _lib.check(_lib.load().otf_repo_rank_many(self._handle, _lib.ptr(W), W.shape[0], k_eff, _lib.ptr(ids),
                                                      _lib.ptr(sc), C.byref(got), _lib.MEM_HOST, None))
        out = []
        row_of = None
        if self.names is not None:
            row_of = {int(v): i for i, v in enumerate(self.ids)}
        for i, m in enumerate(models):
            names = tuple(self.names[row_of[int(x)]] for x in ids[i]) if row_of is not None else None
            out.append(RankedList(ids[i].copy(), sc[i].copy(), model_version(m), produced_at, names))
        return out

    def rank_published(self, trainer, k: int, produced_at: float = 0.0, model_version: int = 0) -> RankedList:
        """rank(k) under the w ``trainer`` last published (``OnlineTrainer.publish_to``): same
        list as ``rank(trainer.snapshot(), k)``. The publication belongs to the trainer, so
        sessions sharing this repository never rank under each other's weights."""
        n = self.count
        k_eff = max(0, min(int(k), n))
        out_ids = np.empty(k_eff, dtype=np.int64)
        out_sc = np.empty(k_eff, dtype=np.float64)
        out_rows = np.empty(k_eff, dtype=np.int64) if self.names is not None else None
        got = C.c_int64(0)
        _lib.check(_lib.load().otf_repo_rank_published(self._handle, trainer.handle, k_eff, _lib.ptr(out_ids),
                                                       _lib.ptr(out_sc), _lib.ptr(out_rows), C.byref(got)))
        if k_eff == 0:
            return _empty_list(model_version, produced_at, self.names)
        names = tuple(self.names[int(r)] for r in out_rows) if self.names is not None else None
        return RankedList(out_ids, out_sc, model_version, produced_at, names)

    def rank(self, model, k: int, produced_at: float = 0.0) -> RankedList:
        w = self._weights(model)
        n = self.count
        k_eff = max(0, min(int(k), n))
        ver = model_version(model)
        if k_eff == 0:
            return _empty_list(ver, produced_at, self.names)
        # one (3, k) int64 block for ids, float64 score bits and rows: one allocation and one
        # address lookup on the per-query path
        block = np.empty((3, k_eff), dtype=np.int64)
        base = _lib.ptr(block)
        rc = _lib.load().otf_repo_rank(self._handle, _lib.ptr(w), k_eff, base, base + 8 * k_eff,
                                       base + 16 * k_eff if self.names is not None else None, None, _lib.MEM_HOST,
                                       None)
        if rc:
            _lib.check(rc)
        names = tuple(self.names[int(r)] for r in block[2]) if self.names is not None else None
        return RankedList._make(block[0], block[1].view(np.float64), ver, produced_at, names)


__all__ = ["RankedList", "RankerConfig", "Repository", "score_dense", "score_pq", "score_binary", "top_k",
           "LinearModel", "DEFAULT_LIST_SIZE", "DEFAULT_RANK_INTERVAL"]
