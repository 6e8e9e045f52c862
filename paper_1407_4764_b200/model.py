"""LinearModel — the immutable weight snapshot the ranker consumes (reference model.py:20-35)."""

from __future__ import annotations

import dataclasses

import numpy as np

from .errors import ConfigError


@dataclasses.dataclass(frozen=True)
class LinearModel:
    """float64 (d,) read-only weights plus provenance counters (model.py:21-35)."""

    weights: np.ndarray
    iteration: int
    version: int = 0

    def __post_init__(self):
        w = np.ascontiguousarray(self.weights, dtype=np.float64)
        if w.ndim != 1 or w.size == 0:
            raise ConfigError(f"weights must be a non-empty 1-D array, got shape {w.shape}")
        w.setflags(write=False)
        object.__setattr__(self, "weights", w)

    @property
    def dim(self) -> int:
        return self.weights.shape[0]


def as_weights(model) -> np.ndarray:
    """ranker.py:59-60: accept a LinearModel (ours or the reference's) or a bare array."""
    w = model.weights if hasattr(model, "weights") else model
    return np.ascontiguousarray(np.asarray(w), dtype=np.float64)


def model_version(model) -> int:
    return int(getattr(model, "version", 0))
