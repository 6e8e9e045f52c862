"""Multi-rank ranking plumbing on CPU: world_size 2 (and 3) over gloo.

The product backend (GpuShardBackend) runs the local top-k and the merge in CUDA kernels; here a
CPU backend built on the pinned oracle stands in for those two kernels so the collective logic
(w broadcast, padding of short shards, all_gather, exact merge, global row offsets) is checked
against single-process ranking of the whole repository — bit-identical ids and scores.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import otf_oracle as O
from paper_1407_4764_b200.distributed import PAD_BASE, ShardedRepository, shard_bounds


class OracleBackend:
    """Scores are precomputed for the whole repository and sliced per shard: each row's score
    must not depend on its shard (the CUDA kernels guarantee that; numpy's sgemv blocking does
    not), and this backend only stands in for the select / merge steps."""

    def __init__(self, scores, ids, offset):
        self.s, self.ids, self.offset = scores, ids, offset

    def to_device(self, arr):
        return torch.as_tensor(arr)

    def local_topk(self, w_dev, k):
        ids, sc, rows = O.top_k(self.s, k, self.ids)
        n = len(ids)
        out_sc = np.full(k, -np.inf)
        out_ids = PAD_BASE + np.arange(k, dtype=np.int64)
        out_rows = np.full(k, -1, np.int64)
        out_sc[:n], out_ids[:n], out_rows[:n] = sc, ids, rows + self.offset
        return torch.as_tensor(out_sc), torch.as_tensor(out_ids), torch.as_tensor(out_rows)

    def merge_topk(self, sc, ids, rows, k):
        o_ids, o_sc, pos = O.top_k(sc.numpy(), k, ids.numpy())
        return torch.as_tensor(o_sc), torch.as_tensor(o_ids), rows[torch.as_tensor(pos)]

    def to_host(self, t):
        return t.numpy()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, case, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n, d, k, kind, seed = case
        rng = np.random.default_rng(seed)
        x = rng.standard_normal((n, d)).astype(np.float32)
        if kind == "ties":
            x = np.round(x)
        ids = rng.permutation(n * 2)[:n].astype(np.int64)
        names = [f"r{i}" for i in range(n)]
        w_root = rng.standard_normal(d)
        w = w_root if rank == 0 else np.zeros(d)  # root's w must win
        start, stop = shard_bounds(n, world, rank)
        scores = O.score_dense(w_root, x)
        be = OracleBackend(scores[start:stop], ids[start:stop], start)
        repo = ShardedRepository(be, n, d, names=names)
        got = repo.rank(w, k)
        q.put((rank, got.ids.tolist(), got.scores.tolist(), list(got.names)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,case", [
    (2, (1000, 16, 50, "rand", 1)),
    (2, (101, 8, 100, "ties", 2)),     # k > local shard size: padding path
    (3, (10, 4, 10, "rand", 3)),       # k == N, tiny shards
    (2, (3000, 12, 700, "ties", 4)),   # heavy ties across shards: id tie-break
    (3, (500, 6, 1, "rand", 5)),
])
def test_sharded_rank_equals_single_process(world, case):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    n, d, k, kind, seed = case
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((n, d)).astype(np.float32)
    if kind == "ties":
        x = np.round(x)
    ids = rng.permutation(n * 2)[:n].astype(np.int64)
    w = rng.standard_normal(d)
    ref_ids, ref_sc, ref_rows = O.top_k(O.score_dense(w, x), k, ids)
    for rank, got_ids, got_sc, got_names in results:
        assert got_ids == ref_ids.tolist()
        assert got_sc == ref_sc.tolist()
        assert got_names == [f"r{i}" for i in ref_rows]


def test_shard_bounds_cover_rows_once():
    for n in (0, 1, 7, 1000, 1001):
        for world in (1, 2, 3, 8):
            spans = [shard_bounds(n, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1
