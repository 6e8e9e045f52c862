"""Row-sharded ranking over several GPUs — one process per GPU.

The repository is split into contiguous row ranges, one per rank; every row keeps its global
int64 id. A query is
  1. broadcast of w (d float64) from the root rank        — NCCL over NVLink/NVSwitch
  2. local exact top-k on each GPU (score + select kernels) — no collective
  3. all_gather of the k local candidates (score f64, id, global row) per rank
  4. exact merge of the G*k candidates by (-score, id) on the GPU (the same top-k kernel).
Because (-score, id) is a total order and each row's score does not depend on where the row
lives, the merged list is bit-identical to ranking the whole repository on one GPU, at any GPU
count. Ranks with fewer than k rows pad with (-inf, id = PAD_BASE + slot) entries, which sort
after every real entry and are never selected (k_eff <= total rows).

The collective/merge plumbing is backend-agnostic (``ShardBackend``) so the multi-rank logic is
tested on CPU with gloo (tests/test_distributed.py); the product backend is ``GpuShardBackend``.
"""

from __future__ import annotations

import ctypes as C
from typing import Protocol

import numpy as np

from . import _lib
from .errors import ConfigError
from .model import as_weights, model_version
from .ranker import RankedList, Repository

PAD_BASE = 1 << 62


def shard_bounds(n_total: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced row range [start, stop) of `rank` (first n%world ranks get +1)."""
    base, extra = divmod(n_total, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def pack_candidates(sc, ids, rows):
    """3k int64 send block of one rank: float64 score bit patterns, then ids, then global rows."""
    import torch

    return torch.cat((sc.contiguous().view(torch.int64), ids.contiguous(), rows.contiguous()))


def unpack_candidates(gathered, world: int):
    """world*3k gathered blocks -> world*k float64 scores, ids, rows in rank order."""
    import torch

    g = gathered.view(world, 3, -1).transpose(0, 1).reshape(3, -1)
    return g[0].contiguous().view(torch.float64), g[1].contiguous(), g[2].contiguous()


class ShardBackend(Protocol):
    def to_device(self, arr: np.ndarray): ...
    def local_topk(self, w_dev, k: int): ...          # -> (scores f64[k], ids i64[k], rows i64[k]) padded
    def merge_topk(self, scores, ids, rows, k: int): ...  # -> (scores, ids, rows) of k_eff best
    def to_host(self, t) -> np.ndarray: ...


class GpuShardBackend:
    """Device tensors are torch CUDA tensors (allocation + NCCL); all math is our kernels."""

    def __init__(self, local: Repository, row_offset: int):
        import torch

        self.torch = torch
        self.local = local
        self.row_offset = int(row_offset)
        self.device = torch.device("cuda", local.device)
        self._bufs: dict[int, tuple] = {}

    def _stream(self):
        return C.c_void_p(self.torch.cuda.current_stream(self.device).cuda_stream)

    def to_device(self, arr):
        return self.torch.tensor(arr, device=self.device)  # (a copy: the model's w may be read-only)

    def local_topk(self, w_dev, k: int):
        torch = self.torch
        n = self.local.count
        k_loc = min(k, n)
        if k not in self._bufs:
            sc = torch.empty(k, dtype=torch.float64, device=self.device)
            ids = torch.empty(k, dtype=torch.int64, device=self.device)
            rows = torch.empty(k, dtype=torch.int64, device=self.device)
            self._bufs[k] = (sc, ids, rows)
        sc, ids, rows = self._bufs[k]
        if k_loc < k:
            sc[k_loc:].fill_(float("-inf"))
            ids[k_loc:] = torch.arange(PAD_BASE + k_loc, PAD_BASE + k, device=self.device)
            rows[k_loc:].fill_(-1)
        if k_loc > 0:
            got = C.c_int64()
            _lib.check(_lib.load().otf_repo_rank(self.local.handle, _lib.tptr(w_dev), k_loc, _lib.tptr(ids),
                                                 _lib.tptr(sc), _lib.tptr(rows), C.byref(got), _lib.MEM_DEVICE,
                                                 self._stream()))
            if self.row_offset:
                rows[:k_loc] += self.row_offset
        return sc, ids, rows

    def merge_topk(self, scores, ids, rows, k: int):
        torch = self.torch
        n = scores.numel()
        k_eff = min(k, n)
        out_sc = torch.empty(k_eff, dtype=torch.float64, device=self.device)
        out_ids = torch.empty(k_eff, dtype=torch.int64, device=self.device)
        out_pos = torch.empty(k_eff, dtype=torch.int64, device=self.device)
        got = C.c_int64()
        _lib.check(_lib.load().otf_top_k(self.local.device, _lib.tptr(scores), _lib.F64, n, _lib.tptr(ids), k_eff,
                                         _lib.tptr(out_ids), _lib.tptr(out_sc), _lib.tptr(out_pos), C.byref(got),
                                         _lib.MEM_DEVICE, self._stream()))
        return out_sc, out_ids, rows[out_pos]

    def to_host(self, t) -> np.ndarray:
        return t.cpu().numpy()


class ShardedRepository:
    """A repository whose rows are spread over the ranks of a torch.distributed group.

    Every rank constructs one with its local shard; ``rank(model, k)`` is collective (all ranks
    call it) and returns the global RankedList on every rank (``root_only`` skips the host copy
    on non-root ranks).
    """

    def __init__(self, backend, total_rows: int, model_dim: int, group=None, names=None, root: int = 0):
        import torch.distributed as dist

        self.dist = dist
        self.backend = backend
        self.total_rows = int(total_rows)
        self.model_dim = int(model_dim)
        self.group = group
        self.names = names
        self.root = root

    @classmethod
    def from_local(cls, local: Repository, total_rows: int, row_offset: int, group=None, names=None):
        return cls(GpuShardBackend(local, row_offset), total_rows, local.model_dim, group=group, names=names)

    def rank_device(self, w_dev, k: int):
        """Steps 1-4 on device tensors; returns (scores, ids, rows) of the global top-k."""
        dist = self.dist
        world = dist.get_world_size(self.group)
        dist.broadcast(w_dev, src=self.root, group=self.group)
        k_eff = max(0, min(int(k), self.total_rows))
        if k_eff == 0:
            return None
        sc, ids, rows = self.backend.local_topk(w_dev, k_eff)
        if world == 1:
            return sc[:k_eff], ids[:k_eff], rows[:k_eff]
        # ONE all_gather of a packed 3k int64 block per rank: the float64 scores travel as
        # their bit patterns next to the ids and global rows (one collective, not three)
        packed = pack_candidates(sc, ids, rows)
        gathered = packed.new_empty(world * packed.numel())
        dist.all_gather_into_tensor(gathered, packed, group=self.group)
        all_sc, all_ids, all_rows = unpack_candidates(gathered, world)
        return self.backend.merge_topk(all_sc, all_ids, all_rows, k_eff)

    def rank(self, model, k: int, produced_at: float = 0.0, root_only: bool = False) -> RankedList | None:
        w = as_weights(model)
        if w.shape != (self.model_dim,):
            raise ConfigError(f"store dim {self.model_dim} does not match model dim {w.shape[0]}")
        w_dev = self.backend.to_device(np.ascontiguousarray(w, dtype=np.float64))
        out = self.rank_device(w_dev, k)
        ver = model_version(model)
        if out is None:
            return RankedList(np.empty(0, np.int64), np.empty(0, np.float64), ver, produced_at,
                              tuple() if self.names is not None else None)
        if root_only and self.dist.get_rank(self.group) != self.root:
            return None
        sc, ids, rows = (self.backend.to_host(t) for t in out)
        names = tuple(self.names[int(r)] for r in rows) if self.names is not None else None
        return RankedList(ids.astype(np.int64), sc.astype(np.float64), ver, produced_at, names)


class NcclShardGroup:
    """The same collective ranking through the library's own NCCL communicator (otf_group_*).

    One object per rank over that rank's shard. The 128-byte NCCL unique id is created once
    (``NcclShardGroup.unique_id()`` on one rank) and handed to every rank by any channel (e.g.
    ``torch.distributed.broadcast_object_list``). ``rank`` is collective; w is read on ``root``
    only; every rank receives the global RankedList.
    """

    @staticmethod
    def unique_id() -> bytes:
        buf = (C.c_ubyte * 128)()
        _lib.check(_lib.load().otf_group_unique_id(buf))
        return bytes(buf)

    def __init__(self, shard: Repository, uid: bytes, n_ranks: int, rank: int, row_offset: int, total_rows: int,
                 names=None, root: int = 0):
        if len(uid) != 128:
            raise ConfigError("an NCCL unique id is 128 bytes")
        self.shard = shard
        self.row_offset = int(row_offset)
        self.total_rows = int(total_rows)
        self.names = names
        self.root = int(root)
        self.model_dim = shard.model_dim
        buf = (C.c_ubyte * 128).from_buffer_copy(uid)
        h = C.c_void_p()
        _lib.check(_lib.load().otf_group_create(shard.device, int(n_ranks), int(rank), buf, C.byref(h)))
        self._handle = h

    def close(self) -> None:
        h = getattr(self, "_handle", None)
        if h is not None and h.value and _lib._lib is not None:
            _lib._lib.otf_group_destroy(h)
        self._handle = None

    def __del__(self):
        self.close()

    def rank(self, model, k: int, produced_at: float = 0.0) -> RankedList:
        w = np.ascontiguousarray(as_weights(model), dtype=np.float64)
        if w.shape != (self.model_dim,):
            raise ConfigError(f"store dim {self.model_dim} does not match model dim {w.shape[0]}")
        k_eff = max(0, min(int(k), self.total_rows))
        ids = np.empty(k_eff, np.int64)
        sc = np.empty(k_eff, np.float64)
        rows = np.empty(k_eff, np.int64)
        got = C.c_int64()
        _lib.check(_lib.load().otf_group_rank(self._handle, self.shard.handle, _lib.ptr(w), self.root, self.row_offset,
                                              self.total_rows, int(k), _lib.ptr(ids), _lib.ptr(sc), _lib.ptr(rows),
                                              C.byref(got), _lib.MEM_HOST, None))
        names = tuple(self.names[int(r)] for r in rows) if self.names is not None else None
        return RankedList(ids, sc, model_version(model), produced_at, names)

    def rank_device(self, w_dev, k: int, stream=None):
        """Device tensors in and out (torch): returns (scores, ids, global rows) on this GPU."""
        import torch

        k_eff = max(0, min(int(k), self.total_rows))
        dev = w_dev.device
        sc = torch.empty(k_eff, dtype=torch.float64, device=dev)
        ids = torch.empty(k_eff, dtype=torch.int64, device=dev)
        rows = torch.empty(k_eff, dtype=torch.int64, device=dev)
        if k_eff:
            st = stream if stream is not None else torch.cuda.current_stream(dev)
            got = C.c_int64()
            _lib.check(_lib.load().otf_group_rank(self._handle, self.shard.handle, _lib.tptr(w_dev), self.root,
                                                  self.row_offset, self.total_rows, int(k), _lib.tptr(ids),
                                                  _lib.tptr(sc), _lib.tptr(rows), C.byref(got), _lib.MEM_DEVICE,
                                                  C.c_void_p(st.cuda_stream)))
        return sc, ids, rows
