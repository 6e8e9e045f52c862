"""FeatureStore — the dense repository input layout (reference store.py:56-136).

A read-only (count, dim) float32 C-contiguous matrix with unique non-negative int64 ids and
optional names. ``Repository.dense`` accepts this class or the reference's own FeatureStore
(anything with ``.data``, ``.ids``, ``.names``). File IO and synthetic corpora are out of
scope.
"""

from __future__ import annotations

from typing import Iterable

import numpy as np

from .errors import ConfigError, EmptyStoreError


class FeatureStore:
    """Immutable feature matrix with per-row ids and optional names (store.py:56-136)."""

    def __init__(self, data, ids=None, names=None):
        arr = np.ascontiguousarray(data, dtype=np.float32)
        if arr.ndim != 2:
            raise ConfigError(f"feature data must be 2-D, got shape {arr.shape}")
        if arr.shape[0] == 0 or arr.shape[1] == 0:
            raise EmptyStoreError(f"feature store needs at least one row and one column, got shape {arr.shape}")
        arr.setflags(write=False)
        self._data = arr
        if ids is None:
            id_arr = np.arange(arr.shape[0], dtype=np.int64)
        else:
            id_arr = np.ascontiguousarray(ids, dtype=np.int64)
            if id_arr.shape != (arr.shape[0],):
                raise ConfigError(f"ids shape {id_arr.shape} does not match {arr.shape[0]} rows")
            if np.any(id_arr < 0):
                raise ConfigError("ids must be non-negative")
            if np.unique(id_arr).size != id_arr.size:
                raise ConfigError("ids must be unique")
        id_arr.setflags(write=False)
        self._ids = id_arr
        if names is not None and len(names) != arr.shape[0]:
            raise ConfigError(f"names list has {len(names)} entries for {arr.shape[0]} rows")
        self._names = list(names) if names is not None else None

    @property
    def data(self) -> np.ndarray:
        return self._data

    @property
    def ids(self) -> np.ndarray:
        return self._ids

    @property
    def names(self):
        return list(self._names) if self._names is not None else None

    @property
    def count(self) -> int:
        return self._data.shape[0]

    @property
    def dim(self) -> int:
        return self._data.shape[1]

    def subset(self, rows) -> "FeatureStore":
        rows = np.asarray(rows)
        names = [self._names[i] for i in rows] if self._names is not None else None
        return FeatureStore(self._data[rows], self._ids[rows], names)

    def without_ids(self, excluded: Iterable[int]) -> "FeatureStore":
        drop = np.fromiter((int(i) for i in excluded), dtype=np.int64)
        if drop.size == 0:
            return self
        keep = np.flatnonzero(~np.isin(self._ids, drop))
        if keep.size == 0:
            raise EmptyStoreError("exclusion removed every row")
        return self.subset(keep)
