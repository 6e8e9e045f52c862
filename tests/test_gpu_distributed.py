"""The multi-rank rank path with the PRODUCT backend (GpuShardBackend: local top-k and merge in the
CUDA kernels, through the C ABI) in 2 and 3 separate processes, exchanging over gloo.

This pool has one GPU per box, so the ranks share cuda:0; nothing here makes one rank's kernels
wait on another's (each rank's local top-k and merge are its own launches; the collectives are
gloo's host-side exchange), so this checks the process-level plumbing of §8(e) around the real
kernels — w broadcast from the root, short-shard padding, the packed all_gather of (score bits,
id, global row), the exact device merge — against one process ranking the whole repository
(bit-identical ids and scores). NCCL itself only runs in the driver's multi-GPU scaling run.
"""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _data(case):
    n, d, k, kind, seed = case
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((n, d)).astype(np.float32)
    if kind == "ties":
        x = np.round(x)
    return x, rng.standard_normal(d)


def _worker(rank, world, port, case, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist

    import paper_1407_4764_b200 as otf
    from paper_1407_4764_b200.distributed import ShardedRepository, shard_bounds

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        n, d, k, kind, seed = case
        x, w_root = _data(case)
        start, stop = shard_bounds(n, world, rank)
        class Shard:  # the shard's rows with their global ids (the reference store's .data / .ids)
            data, ids = x[start:stop], np.arange(start, stop, dtype=np.int64)

        local = otf.Repository.dense(Shard())
        sharded = ShardedRepository.from_local(local, n, start)
        w = w_root if rank == 0 else np.zeros(d)  # the root's w must win
        got = sharded.rank(otf.LinearModel(w, 1, 1), k)
        sc, ids, rows = sharded.rank_device(torch.as_tensor(w_root, device="cuda"), k)
        q.put((rank, got.ids.tolist(), got.scores.tolist(), rows.cpu().tolist()))
    except Exception as e:  # surfaced by the parent
        q.put((rank, repr(e), None, None))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,case", [
    (2, (200_000, 128, 1000, "rand", 1)),   # 100k rows per rank: the fused paths on each shard
    (2, (1001, 16, 700, "ties", 2)),        # k > a shard: padding; heavy ties across shards
    (3, (30_001, 256, 100, "rand", 3)),
    (3, (10, 4, 10, "rand", 4)),            # k == N, tiny shards
])
def test_gpu_sharded_rank_equals_single_process(otf, world, case):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
    for rank, got_ids, _, _ in results:
        assert not isinstance(got_ids, str), f"rank {rank}: {got_ids}"
    x, w = _data(case)
    k = case[2]
    ref = otf.Repository.dense(x).rank(otf.LinearModel(w, 1, 1), k)
    rows_ref = [int(i) for i in ref.ids]  # default ids are the rows
    for rank, got_ids, got_sc, got_rows in results:
        assert got_ids == ref.ids.tolist()
        assert np.asarray(got_sc).tobytes() == ref.scores.tobytes()
        assert got_rows == rows_ref
    for p in procs:
        assert p.exitcode == 0
