"""Pegasos hinge-loss SGD on the GPU — drop-in for the reference's trainer.py:1-173.

``pegasos_step`` and ``OnlineTrainer`` keep the reference's signatures, sampling and error
types. Sample indices are drawn on the host with the caller's numpy ``Generator`` exactly as
the reference draws them (positives first, then negatives, with replacement,
trainer.py:95-97), so the batch — and ``batch_hook`` — are identical; the update itself
(margins, violators, gradient, shrink, projection; trainer.py:51-71) runs in one CUDA kernel
(csrc/otf_train.cu). ``OnlineTrainer`` keeps the negative pool and w resident in HBM and steps on
its own high-priority stream, so the per-step cost is O(B*d) instead of the reference's
O(pool) float64 conversion (trainer.py:100-102).
"""

from __future__ import annotations

import ctypes as C
import dataclasses
import math
import threading
from typing import Callable

import numpy as np

from . import _lib
from .errors import ConfigError, InsufficientDataError, NotReadyError
from .model import LinearModel

BatchHook = Callable[[np.ndarray, np.ndarray], None]


@dataclasses.dataclass(frozen=True)
class TrainerConfig:
    """trainer.py:31-48."""

    lam: float = 1.0
    batch_size: int = 32
    project: bool = True
    seed: int = 0

    def validate(self) -> None:
        if self.lam <= 0:
            raise ConfigError(f"lam must be positive, got {self.lam}")
        if self.batch_size < 2 or self.batch_size % 2 != 0:
            raise ConfigError(f"batch_size must be an even number >= 2, got {self.batch_size}")


def _step_scalars(step_index: int, lam: float, batch_size: int):
    """The Python-double scalars of trainer.py:61,65,67 (computed exactly as the reference)."""
    eta = 1.0 / (lam * step_index)
    return (1.0 - eta * lam), (eta / batch_size), (1.0 / math.sqrt(lam))


def _pool_array(pool) -> np.ndarray:
    return pool.data if hasattr(pool, "data") and not isinstance(pool, np.ndarray) else np.asarray(pool)


def pegasos_step(weights, step_index, positives, negatives, cfg: TrainerConfig, rng: np.random.Generator,
                 batch_hook: BatchHook | None = None) -> np.ndarray:
    """trainer.py:74-106 — one balanced mini-batch update; returns the new float64 w."""
    cfg.validate()
    if step_index < 1:
        raise ConfigError(f"step_index must be >= 1, got {step_index}")
    pos = _pool_array(positives)
    neg = _pool_array(negatives)
    if len(pos) == 0:
        raise NotReadyError("no positives available yet")
    if len(neg) == 0:
        raise InsufficientDataError("negative pool is empty")
    half = cfg.batch_size // 2
    pos_idx = rng.integers(0, len(pos), size=half)
    neg_idx = rng.integers(0, len(neg), size=half)
    if batch_hook is not None:
        batch_hook(pos_idx, neg_idx)
    # gather the B sampled rows (O(B*d)) into one float64 batch, positives first
    batch = np.empty((2 * half, pos.shape[1]), dtype=np.float64)
    batch[:half] = pos[pos_idx]
    batch[half:] = neg[neg_idx]
    w = np.array(weights, dtype=np.float64, copy=True, order="C")
    if w.shape != (batch.shape[1],):
        raise ConfigError(f"weights shape {w.shape} does not match pool dim {batch.shape[1]}")
    shrink, eob, radius = _step_scalars(step_index, cfg.lam, cfg.batch_size)
    _lib.check(_lib.load().otf_pegasos_step_host(_lib.default_device(), _lib.ptr(w), w.shape[0], _lib.ptr(batch),
                                                 half, shrink, eob, int(bool(cfg.project)), radius))
    return w


class OnlineTrainer:
    """trainer.py:109-173 — single-writer streaming trainer with locked snapshots.

    The negative pool is copied to HBM once; w lives in HBM. ``step(positives)`` samples on
    the host and gathers only the B/2 sampled positive rows; ``step()`` with no argument uses
    the device-resident positive pool filled by ``append_positives`` (the GPU analogue of
    session.py:62-93 PositivePool).
    """

    def __init__(self, dim: int, negatives, cfg: TrainerConfig | None = None, batch_hook: BatchHook | None = None,
                 device: int | None = None):
        self.cfg = cfg if cfg is not None else TrainerConfig()
        self.cfg.validate()
        neg = _pool_array(negatives)
        neg = np.asarray(neg)
        if neg.ndim != 2 or neg.shape[0] == 0:
            raise InsufficientDataError("negative pool must be a non-empty 2-D array")
        if neg.shape[1] != dim:
            raise ConfigError(f"negative pool dim {neg.shape[1]} does not match model dim {dim}")
        # the reference stores OnlineTrainer negatives as float32 whatever their dtype
        # (trainer.py:127: np.asarray(negatives, dtype=np.float32)); pegasos_step then widens the
        # float32 rows to float64 exactly, which the kernel does per sampled row
        self._neg_dtype = _lib.F32
        neg = np.ascontiguousarray(neg, dtype=np.float32)
        self._dim = int(dim)
        self._n_neg = neg.shape[0]
        self._batch_hook = batch_hook
        self._rng = np.random.default_rng(self.cfg.seed)
        self._lock = threading.Lock()
        self._pool_lock = threading.Lock()
        self._n_pos = 0
        self._iteration = 0
        self._version = 0
        self._published_iteration = -1
        self._snap: LinearModel | None = None
        self._device = _lib.default_device() if device is None else device
        h = C.c_void_p()
        _lib.check(_lib.load().otf_trainer_create(self._device, self._dim, _lib.ptr(neg), self._neg_dtype,
                                                  self._n_neg, _lib.MEM_HOST, C.byref(h)))
        self._handle = h

    def __del__(self):
        h = getattr(self, "_handle", None)
        if h is not None and h.value and _lib._lib is not None:
            _lib._lib.otf_trainer_destroy(h)
            self._handle = None

    @property
    def iteration(self) -> int:
        return self._iteration

    @property
    def handle(self) -> C.c_void_p:
        return self._handle

    def append_positives(self, rows) -> int:
        """Append float32 rows to the device positive pool; returns the pool size."""
        arr = np.ascontiguousarray(np.atleast_2d(np.asarray(rows, dtype=np.float32)))
        if arr.shape[1] != self._dim:
            raise ConfigError(f"vector shape {arr.shape[1:]} does not match pool dim {self._dim}")
        _lib.check(_lib.load().otf_trainer_append_positives(self._handle, _lib.ptr(arr), _lib.F32, arr.shape[0],
                                                            _lib.MEM_HOST))
        # the pool size is tracked here, not read back: one library call (one GIL round trip)
        # per append keeps the feeder cheap when a busy Python thread holds the GIL
        with self._pool_lock:
            self._n_pos += arr.shape[0]
            return self._n_pos

    def step(self, positives=None) -> int:
        """trainer.py:145-159 — one update against the given (or the device) positive pool."""
        cfg = self.cfg
        half = cfg.batch_size // 2
        if positives is not None:
            pos = _pool_array(positives)
            pos = np.asarray(pos)
            n_pos = len(pos)
        else:
            n_pos = self._n_pos  # rows whose append has completed (the device pool holds them)
            pos = None
        if n_pos == 0:
            raise NotReadyError("no positives available yet")
        t = self._iteration + 1
        pos_idx = self._rng.integers(0, n_pos, size=half)
        neg_idx = self._rng.integers(0, self._n_neg, size=half)
        if self._batch_hook is not None:
            self._batch_hook(pos_idx, neg_idx)
        shrink, eob, radius = _step_scalars(t, cfg.lam, cfg.batch_size)
        pidx = np.ascontiguousarray(pos_idx, dtype=np.int64)
        nidx = np.ascontiguousarray(neg_idx, dtype=np.int64)
        with self._lock:  # (w, iteration) change together, as under trainer.py:156-159
            if pos is not None:
                pdt = _lib.F64 if pos.dtype == np.float64 else _lib.F32
                parr = np.ascontiguousarray(pos, dtype=np.float64 if pdt == _lib.F64 else np.float32)
                if parr.ndim != 2 or parr.shape[1] != self._dim:
                    raise ConfigError(f"positive pool shape {parr.shape} does not match dim {self._dim}")
                _lib.check(_lib.load().otf_trainer_step(self._handle, _lib.ptr(parr), pdt, n_pos, _lib.ptr(pidx),
                                                        _lib.ptr(nidx), half, shrink, eob, int(bool(cfg.project)),
                                                        radius))
            else:
                _lib.check(_lib.load().otf_trainer_step(self._handle, None, _lib.F32, n_pos, _lib.ptr(pidx),
                                                        _lib.ptr(nidx), half, shrink, eob, int(bool(cfg.project)),
                                                        radius))
            self._iteration = t
            return self._iteration

    def weights_device_ptr(self) -> int:
        """Device address of the live float64 w (for zero-copy ranking on the same GPU)."""
        p = C.c_void_p()
        _lib.check(_lib.load().otf_trainer_weights_ptr(self._handle, C.byref(p)))
        return int(p.value or 0)

    def _sync_version(self) -> None:
        """(under _lock) version bumps only when the iterate moved (trainer.py:167-173)."""
        if self._iteration != self._published_iteration:
            self._version += 1
            self._published_iteration = self._iteration
            self._snap = None

    def snapshot(self) -> LinearModel:
        """trainer.py:161-173 — immutable copy; version bumps only when the iterate moved."""
        with self._lock:
            if self._iteration == 0:
                raise NotReadyError("no training step has run yet")
            self._sync_version()
            if self._snap is None:
                w = np.empty(self._dim, dtype=np.float64)
                _lib.check(_lib.load().otf_trainer_weights(self._handle, _lib.ptr(w), _lib.MEM_HOST))
                self._snap = LinearModel(w, self._iteration, self._version)
            return LinearModel(self._snap.weights.copy(), self._snap.iteration, self._snap.version)

    def publish_to(self, repository) -> tuple[int, int]:
        """The device-side snapshot: w goes straight into ``repository``'s ranking buffer (one
        device copy + CUDA event, no host round trip); returns (iteration, version) with the
        versioning of snapshot(). Rank it with ``repository.rank_published``."""
        with self._lock:
            if self._iteration == 0:
                raise NotReadyError("no training step has run yet")
            self._sync_version()
            _lib.check(_lib.load().otf_trainer_publish(self._handle, repository.handle))
            return self._iteration, self._version


# -- fixed-set training (trainer.py:176-257) ------------------------------------------------------


@dataclasses.dataclass(frozen=True)
class BatchTrainConfig:
    """trainer.py:178-194 — C-parameterised regularisation and epoch budget."""

    c: float = 0.25
    batch_size: int = 32
    epochs: int = 60
    project: bool = True
    seed: int = 0

    def validate(self) -> None:
        if self.c <= 0:
            raise ConfigError(f"c must be positive, got {self.c}")
        if self.batch_size < 1:
            raise ConfigError(f"batch_size must be >= 1, got {self.batch_size}")
        if self.epochs < 1:
            raise ConfigError(f"epochs must be >= 1, got {self.epochs}")


def _pooled(positives, negatives):
    pos = np.asarray(_pool_array(positives))
    neg = np.asarray(_pool_array(negatives))
    if len(pos) == 0 or len(neg) == 0:
        raise InsufficientDataError("both classes need at least one example")
    if pos.shape[1] != neg.shape[1]:
        raise ConfigError(f"dim mismatch: positives {pos.shape[1]}, negatives {neg.shape[1]}")
    # the reference converts both pools to float64 (exact for float32 inputs); keep float32 rows
    # in float32 on the device when both pools are float32 (half the HBM), else float64
    if pos.dtype == np.float32 and neg.dtype == np.float32:
        return np.ascontiguousarray(np.concatenate([pos, neg])), _lib.F32, len(pos)
    feats = np.concatenate([pos.astype(np.float64), neg.astype(np.float64)])
    return np.ascontiguousarray(feats), _lib.F64, len(pos)


def hinge_objective(weights, features, labels, lam: float) -> float:
    """trainer.py:197-201 — lam/2 |w|^2 + mean hinge loss, on the GPU.

    ``labels`` must be +1 for a leading block of rows and -1 for the rest (the layout
    train_batch uses); other label layouts are reordered on the host first.
    """
    x = np.asarray(features)
    y = np.asarray(labels)
    order = np.argsort(-y, kind="stable")  # +1 rows first, original order within each class
    x = np.ascontiguousarray(x[order])
    n_pos = int(np.count_nonzero(y > 0))
    dt = _lib.F32 if x.dtype == np.float32 else _lib.F64
    x = np.ascontiguousarray(x, dtype=np.float32 if dt == _lib.F32 else np.float64)
    w = np.ascontiguousarray(weights, dtype=np.float64)
    out = np.empty(1, dtype=np.float64)
    _lib.check(_lib.load().otf_hinge_objective(_lib.default_device(), _lib.ptr(x), dt, n_pos, x.shape[0], x.shape[1],
                                               _lib.ptr(w), float(lam), _lib.ptr(out), _lib.MEM_HOST, None))
    return float(out[0])


def train_batch(positives, negatives, cfg: BatchTrainConfig | None = None, objective_history=None) -> LinearModel:
    """trainer.py:204-257 — fixed-set SVM fit; one persistent CUDA CTA runs every step."""
    cfg = cfg if cfg is not None else BatchTrainConfig()
    cfg.validate()
    feats, dt, n_pos = _pooled(positives, negatives)
    n, d = feats.shape
    lam = 1.0 / (cfg.c * n)
    batch_size = min(cfg.batch_size, n)
    steps_per_epoch = math.ceil(n / batch_size)
    total_steps = cfg.epochs * steps_per_epoch
    tail_len = max(1, total_steps // 4)
    tail_start = total_steps - tail_len
    rng = np.random.default_rng(cfg.seed)
    # the reference draws rng.integers(0, n, size=batch_size) once per step (trainer.py:243)
    idx = np.empty((total_steps, batch_size), dtype=np.int64)
    for t in range(total_steps):
        idx[t] = rng.integers(0, n, size=batch_size)
    w = np.empty(d, dtype=np.float64)
    hist = np.empty(total_steps // steps_per_epoch + 1, dtype=np.float64)
    _lib.check(_lib.load().otf_train_batch(_lib.default_device(), _lib.ptr(feats), dt, n_pos, n, d, _lib.ptr(idx),
                                           total_steps, batch_size, steps_per_epoch, tail_start, tail_len, lam,
                                           int(bool(cfg.project)), _lib.ptr(w), _lib.ptr(hist), _lib.MEM_HOST, None))
    if objective_history is not None:
        objective_history.extend(float(v) for v in hist[:-1])
    return LinearModel(w, total_steps)
