"""Per-step timing breakdown of the rank path (diagnostic, not the bench)."""
import ctypes as C
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
from paper_1407_4764_b200 import _lib  # noqa: E402

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
dev = torch.device("cuda", 0)
repo, keep, _ = bench.make_repository(cfg, 0, 1, 0)
lib = _lib.load()
k = cfg["k"]
w = torch.as_tensor(np.random.default_rng(1).standard_normal(repo.model_dim), device=dev)
ids = torch.empty(k, dtype=torch.int64, device=dev)
sc = torch.empty(k, dtype=torch.float64, device=dev)
rows = torch.empty(k, dtype=torch.int64, device=dev)
buf = torch.empty(repo.count, dtype=torch.float64, device=dev)
got = C.c_int64()


def timed(name, fn, reps=50, stream=None):
    s = stream or torch.cuda.current_stream()
    sp = C.c_void_p(s.cuda_stream)
    for _ in range(3):
        fn(sp)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(s)
    for _ in range(reps):
        fn(sp)
    e1.record(s)
    torch.cuda.synchronize()
    host = (time.perf_counter() - t0) / reps * 1e3
    print(f"{name:40s} device {e0.elapsed_time(e1) / reps:8.4f} ms/iter   host {host:8.4f} ms/iter")


def score(sp):
    _lib.check(lib.otf_repo_score(repo.handle, _lib.tptr(w), _lib.tptr(buf), _lib.MEM_DEVICE, sp))


def rank(sp):
    _lib.check(lib.otf_repo_rank(repo.handle, _lib.tptr(w), k, _lib.tptr(ids), _lib.tptr(sc), _lib.tptr(rows),
                                 C.byref(got), _lib.MEM_DEVICE, sp))


def rank_graph(sp):
    _lib.check(lib.otf_repo_rank_graph(repo.handle, _lib.tptr(w), k, _lib.tptr(ids), _lib.tptr(sc), _lib.tptr(rows), sp))


timed("score only (default stream)", score)
timed("rank (default stream)", rank)
side = torch.cuda.Stream()
with torch.cuda.stream(side):
    timed("score only (side stream)", score, stream=side)
    timed("rank (side stream)", rank, stream=side)
    timed("rank via CUDA graph (side stream)", rank_graph, stream=side)
