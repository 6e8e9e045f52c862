#!/usr/bin/env python
"""bench.py — dataset images scored + exactly ranked per second on B200 (BASELINE.json metric).

One "step" = one query of the on-the-fly ranker: w (float64, resident) -> score every row of the
GPU-resident repository with the linear SVM -> exact top-k by (-score, id) -> (N>1: NCCL
all_gather of the k local candidates + exact merge on the GPU). At N=1 the default workload is
BASELINE.json configs[1] (C2: 1M x 2048-D float32 rows, top-1000); under torchrun every rank holds
its own shard of that size (weak scaling, rows sharded by image, w broadcast from rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2|c1|c3|c4|c5a] [--impl reference]

Rank 0 prints ONE JSON line. `value` is device-timed (CUDA events on the launching stream, max
over ranks); `e2e` is the same metric through the public API (Repository.rank /
ShardedRepository.rank with host w in, host RankedList out, copies inside the timed region);
`roofline` is the dominant (scoring) kernel's algorithmic HBM bytes / its event-timed duration;
`cpu_baseline` is the oracle port (numpy, the reference's own arithmetic) on this host's cores.
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

L2_BYTES = 126 * 1024 * 1024

CONFIGS = {
    "c2": dict(kind="dense", rows=1_000_000, dim=2048, k=1000,
               workload="C2: 1M x 2048-D fp32 features per GPU, single-query linear-SVM score + exact top-1000"),
    "c1": dict(kind="dense", rows=1_000_000, dim=128, k=1000,
               workload="C1: 1M x 128-D fp32 features per GPU, single-query linear-SVM score + exact top-1000",
               # PAPER.md:751-752 (GTX Titan): score 1M CNN-128 features ~0.01 s + rank ~0.002 s
               published=1_000_000 / 0.012),
    "c4": dict(kind="dense", rows=6_250_000, dim=2048, k=1000, train=True,
               workload="C4: 6.25M x 2048-D fp32 rows per GPU (50M over 8 GPUs), score + top-1000 + NCCL merge, "
                        "Pegasos training concurrent with ranking (rank 0, own stream)"),
    "c3": dict(kind="pq", rows=10_000_000, dim=16, k=1000, subdim=8,
               workload="C3: 10M PQ codes per GPU (16 sub-quantizers x 256 centroids, 128-D), LUT score + top-1000"),
    "c3e": dict(kind="pqenc", rows=10_000_000, dim=16, subdim=8, k=0,
                workload="C3 ingest (SURVEY.md §8f): pq_encode of 10M x 128-D fp32 vectors per GPU "
                         "under a 16 x 256 x 8 codebook (nearest centroid per block, float64)"),
    "c3k": dict(kind="pqlearn", rows=50_000, dim=16, subdim=8, k=256, iterations=8,
                workload="C3 codebook (SURVEY.md §8f): learn_pq_codebook on 50k x 128-D fp32 training vectors, "
                         "16 blocks x 256 centroids x 8 dims, 8 Lloyd iterations"),
    "c5a": dict(kind="binary", rows=100_000_000, dim=2048, k=1000,
                workload="C5a: 100M x 2048-bit packed binary codes per GPU, score + top-1000"),
    "c5b": dict(kind="multi", rows=10_000_000, dim=4096, k=1000, n_cls=64,
                workload="C5b: 64 concurrent classifiers over 10M x 4096-D fp32 rows per GPU "
                         "(tcgen05 skinny GEMM, 3 split FP16 products) + exact top-1000 per classifier"),
}


# the scoring kernel of the rank path, per repository kind (otf_repo_time_rank_scan times it)
SCAN_KERNEL = {"dense": "dense_score_fast", "pq": "pq_scan16_f32bins (float32 screening, exact bins)",
               "binary": "bin_score_bytes (2 slice launches)"}


def load_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d.get("hbm_gbs", 6650.0)), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def row_bytes(cfg) -> int:
    if cfg["kind"] in ("dense", "multi"):
        return 4 * cfg["dim"]
    if cfg["kind"] == "pq":
        return cfg["dim"]
    return cfg["dim"] // 8


def metric_unit(cfg) -> tuple[str, str]:
    if cfg["kind"] == "pqlearn":
        return "PQ codebook learning time (learn_pq_codebook)", "ms"
    if cfg["kind"] == "pqenc":
        return "vectors PQ-encoded/sec", "vectors/s"
    if cfg["kind"] == "multi":
        return "dataset images scored+ranked/sec", "image-classifier pairs/s"
    return "dataset images scored+ranked/sec", "images/s"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled while the timed region runs."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except FileNotFoundError:
            self.proc = None
        time.sleep(0.15)
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc is not None:
            time.sleep(0.12)
            self.proc.terminate()
            out, _ = self.proc.communicate(timeout=10)
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self):
        sm, mx, pw, reasons = [], [], [], set()
        for line in getattr(self, "lines", []):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            try:
                pw.append(float(parts[2]))
            except ValueError:
                pass
            for name, val in zip(self.NAMES, parts[3:7]):
                if val.lower() == "active":
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(mx)), "reasons": sorted(reasons),
                "samples": len(sm), "power_w": float(np.median(pw)) if pw else None}


# ---------------------------------------------------------------------------------------------
# reference arm / CPU baseline: the oracle port (numpy = the reference's own arithmetic)


def cpu_sample(cfg, seed=1234):
    """A bounded host sample of the workload and its oracle ranker (sized to ~0.05-0.2 s/query)."""
    sys.path.insert(0, str(ROOT / "oracle"))
    import otf_oracle as O

    rng = np.random.default_rng(seed)
    kind, dim, k = cfg["kind"], cfg["dim"], cfg["k"]
    if kind in ("dense", "multi"):
        rows = max(20_000, min(cfg["rows"], (1 << 30) // (4 * dim)))  # <= 1 GiB of features
        x = rng.standard_normal((rows, dim), dtype=np.float32)
        x /= np.linalg.norm(x, axis=1, keepdims=True)
        if kind == "multi":  # the reference API has one score_dense + top_k per classifier
            W = rng.standard_normal((cfg["n_cls"], dim))
            fn = lambda: [O.top_k(O.score_dense(w, x), k) for w in W]
            desc = (f"{cfg['n_cls']} classifiers x {rows} x {dim}-D fp32 rows (one score_dense + top_k per "
                    "classifier, ranker.py:63-143); unit = image-classifier pairs")
            return rows * cfg["n_cls"], fn, desc
        w = rng.standard_normal(dim)
        fn = lambda: O.top_k(O.score_dense(w, x), k)
        desc = f"{rows} x {dim}-D fp32 rows (score_dense + top_k, ranker.py:63-143)"
    elif kind == "pqlearn":
        x = rng.standard_normal((cfg["rows"], dim * cfg["subdim"]), dtype=np.float32)
        x /= np.linalg.norm(x, axis=1, keepdims=True)
        blocks = 2  # of dim; the per-block work is identical, the value is scaled to all blocks
        sub = x[:, :blocks * cfg["subdim"]]
        fn = lambda: O.learn_pq_codebook(sub, cfg["subdim"], cfg["k"], cfg["iterations"], 5)
        desc = (f"learn_pq_codebook on {cfg['rows']} x {blocks * cfg['subdim']}-D ({blocks} of {dim} blocks, "
                f"{cfg['k']} centroids, {cfg['iterations']} iterations, pq.py:116-203); value scaled x{dim // blocks}")
        return dim / blocks, fn, desc
    elif kind == "pqenc":
        rows = min(cfg["rows"], 40_000)
        cents = rng.standard_normal((dim, 256, cfg["subdim"])).astype(np.float32)
        x = rng.standard_normal((rows, dim * cfg["subdim"]), dtype=np.float32)
        x /= np.linalg.norm(x, axis=1, keepdims=True)
        fn = lambda: O.pq_encode(cents, x)
        desc = f"pq_encode of {rows} x {dim * cfg['subdim']}-D fp32 vectors, {dim} x 256 x {cfg['subdim']} codebook (pq.py:206-230)"
    elif kind == "pq":
        rows = min(cfg["rows"], 2_000_000)
        cents = rng.standard_normal((dim, 256, cfg["subdim"])).astype(np.float32)
        codes = rng.integers(0, 256, (rows, dim), dtype=np.uint8)
        w = rng.standard_normal(dim * cfg["subdim"])
        fn = lambda: O.top_k(O.score_pq(w, cents, codes), k)
        desc = f"{rows} PQ codes x {dim} blocks (build_score_lut + score_codes + top_k, pq.py:248-276)"
    else:
        rows = min(cfg["rows"], 100_000)
        codes = rng.integers(0, 256, (rows, dim // 8), dtype=np.uint8)
        w = rng.standard_normal(dim)
        fn = lambda: O.top_k(O.score_binary(w, codes, dim), k)
        desc = f"{rows} x {dim}-bit codes (score_binary + top_k, ranker.py:78-143)"
    return rows, fn, desc


def cpu_threads() -> int:
    try:
        from threadpoolctl import threadpool_info

        n = [i.get("num_threads") for i in threadpool_info() if i.get("internal_api") == "openblas"]
        if n and n[0]:
            return int(n[0])
    except Exception:
        pass
    return os.cpu_count() or 1


def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    rows, fn, desc = cpu_sample(cfg)
    for _ in range(max(args.warmup, 1)):
        fn()
    times = []
    t_end = time.perf_counter() + 240.0
    for _ in range(args.steps):
        t0 = time.perf_counter()
        fn()
        times.append(time.perf_counter() - t0)
        if time.perf_counter() > t_end:
            break
    per = float(np.mean(times))
    value = rows / per
    metric, unit = metric_unit(cfg)
    if cfg["kind"] == "pqlearn":  # time-like: ms for the whole codebook (rows = block scale factor)
        value = per * rows * 1e3
    line = {
        "impl": "reference", "metric": metric, "value": value, "unit": unit,
        "n_gpus": args.gpus, "steps": len(times), "warmup": args.warmup, "ms_per_step": per * 1e3,
        "higher_is_better": cfg["kind"] != "pqlearn", "scaling": "weak", "vs_baseline": None,
        "dtype": "f32" if cfg["kind"] not in ("pq", "pqlearn") else "f64",
        "data": "synthetic", "config": {"workload": cfg["workload"], "k": cfg["k"], "sample_rows": rows},
        "cpu_baseline": {"value": value, "unit": unit, "cores": cpu_threads(), "kind": "port",
                         "sample": desc + " on host cores; the reference itself (pure numpy) cannot travel to the GPU box"},
        "e2e": {"value": value, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------------------------
# GPU arm


def make_repository(cfg, rank, world, device, seed=20260418):
    import torch

    import paper_1407_4764_b200 as otf

    dev = torch.device("cuda", device)
    n = cfg["rows"]
    start = rank * n  # weak scaling: every rank holds its own n rows; global ids are disjoint
    g = torch.Generator(device=dev)
    g.manual_seed(seed + 7919 * rank)
    keep = {}
    if cfg["kind"] in ("dense", "multi"):
        d = cfg["dim"]
        x = torch.empty((n, d), dtype=torch.float32, device=dev)
        chunk = max(1, (1 << 28) // d)
        for s in range(0, n, chunk):
            v = x[s:s + chunk]
            v.normal_(generator=g)
            v /= v.norm(dim=1, keepdim=True)
        keep["x"] = x
        repo = otf.Repository.from_device("dense", x.data_ptr(), n, d, id_base=start)
    elif cfg["kind"] == "pq":
        m, q = cfg["dim"], cfg["subdim"]
        codes = torch.randint(0, 256, (n, m), dtype=torch.uint8, device=dev, generator=g)
        cents = np.random.default_rng(seed).standard_normal((m, 256, q)).astype(np.float32)
        keep["codes"] = codes
        repo = otf.Repository.from_device("pq", codes.data_ptr(), n, m, id_base=start,
                                          codebook=otf.PQCodebook(cents))
    else:
        bits = cfg["dim"]
        codes = torch.empty((n, bits // 8), dtype=torch.uint8, device=dev)
        chunk = 1 << 24
        for s in range(0, n, chunk):
            codes[s:s + chunk].random_(0, 256, generator=g)
        keep["codes"] = codes
        repo = otf.Repository.from_device("binary", codes.data_ptr(), n, bits, id_base=start)
    torch.cuda.synchronize(dev)
    return repo, keep, start


class ConcurrentTrainer:
    """Pegasos steps in a background thread while the ranking steps are timed (C4: "SGD training
    concurrent with ranking"). The trainer (the package's OnlineTrainer: 16 384 fixed negatives,
    200 positives in its device pool, batch 32) launches on its own high-priority stream; ctypes
    releases the GIL, so its steps interleave with the ranking launches of the main thread."""

    def __init__(self, dim, device):
        import threading

        from paper_1407_4764_b200.trainer import OnlineTrainer, TrainerConfig

        rng = np.random.default_rng(7)
        neg = rng.standard_normal((16_384, dim)).astype(np.float32)
        neg /= np.linalg.norm(neg, axis=1, keepdims=True)
        pos = rng.standard_normal((200, dim)).astype(np.float32) + 0.5
        pos /= np.linalg.norm(pos, axis=1, keepdims=True)
        self.cfg = TrainerConfig(lam=1e-3, batch_size=32, seed=3)
        self.tr = OnlineTrainer(dim, neg, self.cfg, device=device)
        self.tr.append_positives(pos)
        self.steps = 0
        self._stop = threading.Event()
        self._th = threading.Thread(target=self._loop, daemon=True)

    def _loop(self):
        while not self._stop.is_set():
            self.tr.step()
            self.steps += 1

    def start(self):
        self._th.start()

    def mark(self):
        return self.steps, time.perf_counter()

    def stop(self, m0, m1):
        self._stop.set()
        self._th.join()
        steps = m1[0] - m0[0]
        secs = max(m1[1] - m0[1], 1e-9)
        return {"concurrent": True, "trainer_steps_in_timed_region": int(steps),
                "trainer_steps_per_s": steps / secs, "batch": self.cfg.batch_size, "negatives": 16_384,
                "positives": 200, "where": "rank 0, OnlineTrainer on its own high-priority stream",
                "final_iteration": int(self.tr.iteration)}


def run_gpu(args, cfg):
    import torch
    import torch.distributed as dist

    import paper_1407_4764_b200 as otf
    from paper_1407_4764_b200 import _lib
    from paper_1407_4764_b200.distributed import ShardedRepository

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    otf.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    repo, keep, start = make_repository(cfg, rank, world, local)
    n_local = repo.count
    k = cfg["k"]
    total_rows = n_local * world
    dim = repo.model_dim
    w = np.random.default_rng(99).standard_normal(dim)
    w_dev = torch.as_tensor(w, device=dev)
    stream = torch.cuda.current_stream(dev)
    sp = C.c_void_p(stream.cuda_stream)
    lib = _lib.load()
    multi = cfg["kind"] == "multi"
    n_cls = cfg.get("n_cls", 1)  # results per image (classifiers scored together)
    if multi:
        Wm = np.random.default_rng(99).standard_normal((n_cls, dim))
        W_dev = torch.as_tensor(Wm, device=dev)
        m_ids = torch.empty((n_cls, k), dtype=torch.int64, device=dev)
        m_sc = torch.empty((n_cls, k), dtype=torch.float64, device=dev)
        m_got = C.c_int64()

    if multi:
        if world > 1:
            # weak scaling: every rank scores its own rows under all classifiers; per classifier
            # the k local candidates of every rank are all-gathered and merged exactly
            g_sc = torch.empty((world, n_cls, k), dtype=torch.float64, device=dev)
            g_ids = torch.empty((world, n_cls, k), dtype=torch.int64, device=dev)
            f_ids = torch.empty((n_cls, k), dtype=torch.int64, device=dev)
            f_sc = torch.empty((n_cls, k), dtype=torch.float64, device=dev)
            f_got = C.c_int64()

        def step():
            _lib.check(lib.otf_repo_rank_many(repo.handle, _lib.tptr(W_dev), n_cls, k, _lib.tptr(m_ids),
                                              _lib.tptr(m_sc), C.byref(m_got), _lib.MEM_DEVICE, sp))
            if world > 1:
                dist.all_gather_into_tensor(g_sc, m_sc)
                dist.all_gather_into_tensor(g_ids, m_ids)
                c_sc = g_sc.transpose(0, 1).contiguous()    # (n_cls, world * k)
                c_ids = g_ids.transpose(0, 1).contiguous()
                for c in range(n_cls):
                    _lib.check(lib.otf_top_k(local, _lib.tptr(c_sc[c]), _lib.F64, world * k, _lib.tptr(c_ids[c]), k,
                                             _lib.tptr(f_ids[c]), _lib.tptr(f_sc[c]), None, C.byref(f_got),
                                             _lib.MEM_DEVICE, sp))
    elif world > 1 and args.group == "native":
        # the library's own NCCL communicator (otf_group_*); the unique id travels over torch
        from paper_1407_4764_b200.distributed import NcclShardGroup

        uid = [NcclShardGroup.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        sharded = NcclShardGroup(repo, uid[0], world, rank, start, total_rows)
        step = lambda: sharded.rank_device(w_dev, k)
    elif world > 1:
        sharded = ShardedRepository.from_local(repo, total_rows, start)
        step = lambda: sharded.rank_device(w_dev, k)
    else:
        o_ids = torch.empty(k, dtype=torch.int64, device=dev)
        o_sc = torch.empty(k, dtype=torch.float64, device=dev)
        o_rows = torch.empty(k, dtype=torch.int64, device=dev)
        got = C.c_int64()

        if os.environ.get("OTF_BENCH_NO_GRAPH"):
            def step():
                _lib.check(lib.otf_repo_rank(repo.handle, _lib.tptr(w_dev), k, _lib.tptr(o_ids), _lib.tptr(o_sc),
                                             _lib.tptr(o_rows), C.byref(got), _lib.MEM_DEVICE, sp))
        else:
            # the live ranker's path (session.rank_tick): the query's kernels replayed from the
            # repository's cached CUDA graph (no per-launch host work between the kernels)
            def step():
                _lib.check(lib.otf_repo_rank_graph(repo.handle, _lib.tptr(w_dev), k, _lib.tptr(o_ids),
                                                   _lib.tptr(o_sc), _lib.tptr(o_rows), sp))

    payload = n_local * row_bytes(cfg)
    flush = payload < 4 * L2_BYTES
    scratch = torch.empty(2 * L2_BYTES // 4, dtype=torch.float32, device=dev) if flush else None

    def barrier():
        if world > 1:
            dist.barrier()

    train_on = cfg.get("train", False) if args.train is None else args.train
    trainer = ConcurrentTrainer(dim, local) if train_on and rank == 0 else None
    if trainer:
        trainer.start()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)

    # ---- device-timed region: K steps, per-step CUDA events on the launching stream ----------
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    launches0 = _lib.launch_count()
    barrier()
    torch.cuda.synchronize(dev)
    t_mark0 = trainer.mark() if trainer else None
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            if flush:
                scratch.add_(1.0)  # evict the repository from L2 between timed steps (not timed)
            starts[i].record(stream)
            step()
            ends[i].record(stream)
        torch.cuda.synchronize(dev)
    t_mark1 = trainer.mark() if trainer else None
    barrier()
    launches = _lib.launch_count() - launches0
    # the trainer ran beside the timed ranking steps; the kernel-alone and e2e legs run without it
    training = trainer.stop(t_mark0, t_mark1) if trainer else None
    if training:
        training["trainer_launches_in_gpu_launches"] = training["trainer_steps_in_timed_region"]
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    ms = float(np.sum(step_ms)) / args.steps
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        lt = torch.tensor([launches], device=dev, dtype=torch.int64)
        dist.all_reduce(lt)
        launches = int(lt.item())
    value = total_rows * n_cls / (ms / 1e3)

    # ---- dominant kernel (scoring) alone, event-timed: roofline ---------------------------
    score_buf = torch.empty(n_local * n_cls, dtype=torch.float64 if cfg["kind"] == "pq" else torch.float32,
                            device=dev)
    reps = max(5, min(50, args.steps))
    ks, ke = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    kms = []
    kt = C.c_float(0.0)
    for _ in range(reps):
        if flush:
            scratch.add_(1.0)
        if multi:
            ks.record(stream)
            _lib.check(lib.otf_repo_score_many(repo.handle, _lib.tptr(W_dev), n_cls, _lib.tptr(score_buf),
                                               _lib.MEM_DEVICE, sp))
            ke.record(stream)
            torch.cuda.synchronize(dev)
            kms.append(ks.elapsed_time(ke))
        else:
            # the rank path's own scoring kernel (PQ: the float32-screening bins scan), event-timed
            # around its launch on this stream inside the library
            torch.cuda.synchronize(dev)
            _lib.check(lib.otf_repo_time_rank_scan(repo.handle, _lib.tptr(w_dev), C.byref(kt), sp))
            kms.append(float(kt.value))
    kern_ms = float(np.mean(kms))
    peak, peak_src = load_peaks()
    achieved = payload / (kern_ms / 1e3) / 1e9
    traffic = None
    prof = ROOT / "profiles" / f"ncu_{args.config}_summary.json"
    if prof.exists():
        try:
            traffic = json.loads(prof.read_text()).get("dram_bytes_per_launch")
        except Exception:
            traffic = None

    # ---- end to end through the public API (host w in, host RankedList out) ---------------
    e2e_steps = max(3, min(args.steps, 200))
    model = otf.LinearModel(w, 1, 1)
    if multi and world > 1:
        W_pin = torch.from_numpy(Wm).pin_memory()

        def api():  # host W in (pinned H2D), exact global lists out (D2H) on every rank
            W_dev.copy_(W_pin, non_blocking=True)
            step()
            return f_ids.cpu(), f_sc.cpu()
    elif multi:
        models = [otf.LinearModel(wc, 1, 1) for wc in Wm]
        api = lambda: repo.rank_many(models, k)
    elif world > 1 and args.group == "native":
        api = lambda: sharded.rank(model, k)
    elif world > 1:
        api = lambda: sharded.rank(model, k, root_only=True)
    else:
        api = lambda: repo.rank(model, k)
    for _ in range(3):
        api()
    barrier()
    torch.cuda.synchronize(dev)
    e2e_t = []
    for _ in range(e2e_steps):
        if flush:
            scratch.add_(1.0)
            torch.cuda.synchronize(dev)
        barrier()
        t0 = time.perf_counter()
        api()
        e2e_t.append(time.perf_counter() - t0)
    e2e_s = float(np.mean(e2e_t))
    if world > 1:
        t = torch.tensor([e2e_s], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e_val = total_rows * n_cls / e2e_s
    unit = "image-classifier pairs/s" if multi else "images/s"

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        rows, fn, desc = cpu_sample(cfg)
        fn()
        tt = []
        for _ in range(3):
            t0 = time.perf_counter()
            fn()
            tt.append(time.perf_counter() - t0)
        cpu = {"value": rows / min(tt), "unit": unit, "cores": cpu_threads(), "kind": "port",
               "sample": desc + ", oracle port (numpy) best of 3 on this host"}

    if rank == 0:
        line = {
            "metric": "dataset images scored+ranked/sec",
            "value": value,
            "unit": unit,
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms,
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": (value / cfg["published"]) if cfg.get("published") else None,
            "dtype": {"dense": "f32 (f64 accumulate)", "pq": "f64", "binary": "f32 (f64 accumulate)",
                      "multi": "f32 via tcgen05 (3 split fp16 products, f32 accumulate)"}[cfg["kind"]],
            "data": "synthetic",
            "config": {"workload": cfg["workload"], "rows_per_gpu": n_local, "total_rows": total_rows,
                       "dim_or_blocks_or_bits": cfg["dim"], "k": k, "parallelism": f"dp{world} (rows sharded)", "exchange": (args.group if world > 1 else "none"),
                       "l2": ("L2 flushed between timed steps" if flush else
                              f"inputs ({payload / 1e9:.1f} GB/GPU) larger than L2")},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": (f"multi_score_tc (tcgen05 kind::f16, 3 split products, {n_cls} classifiers; "
                                    f"incl. the W split) over {payload / 1e9:.3f} GB"
                                    if multi else
                                    f"{SCAN_KERNEL[cfg['kind']]} (the rank path's scoring kernel, "
                                    f"otf_repo_time_rank_scan) over {payload / 1e9:.3f} GB"),
                         "kernel_ms": kern_ms, "kernel_share_of_step": kern_ms / ms, "peak_source": peak_src,
                         "frac_of_spec_8tbs": achieved / 8000.0},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_val, "unit": unit, "h2d_bytes_per_step": dim * 8 * n_cls,
                    "d2h_bytes_per_step": k * (16 if multi else 24) * n_cls, "ms_per_query": e2e_s * 1e3},
            "gpu_launches": launches,
            "clocks": clk.summary(),
        }
        if training:
            line["training"] = training
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


# FFMA peak derived from the hardware (no FP32 SIMT peak in MEASURED_PEAKS.json):
# 148 SMs x 128 FP32 lanes x 2 flop x 1.965 GHz
FP32_PEAK_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12


def profile_traffic(config):
    prof = ROOT / "profiles" / f"ncu_{config}_summary.json"
    try:
        return json.loads(prof.read_text()).get("dram_bytes_per_launch")
    except Exception:
        return None


def run_encode(args, cfg):
    """C3 ingest: pq_encode of the whole batch of device-resident vectors per step (one GPU per
    rank, each encodes its own rows). The kernel is FP32-FMA bound (K*Q fused multiply-adds per
    vector and block, float32 screening with a float64 decision), so its roofline is FFMA
    throughput, not HBM."""
    import torch
    import torch.distributed as dist

    import paper_1407_4764_b200 as otf
    from paper_1407_4764_b200 import _lib

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    otf.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    n, M, Q, K = cfg["rows"], cfg["dim"], cfg["subdim"], 256
    dim = M * Q
    g = torch.Generator(device=dev)
    g.manual_seed(4242 + rank)
    x = torch.empty((n, dim), dtype=torch.float32, device=dev)
    for s0 in range(0, n, 1 << 21):
        v = x[s0:s0 + (1 << 21)]
        v.normal_(generator=g)
        v /= v.norm(dim=1, keepdim=True)
    cents_np = np.random.default_rng(99).standard_normal((M, K, Q)).astype(np.float32)
    cents = torch.as_tensor(cents_np, device=dev)
    codes = torch.empty((n, M), dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    sp = C.c_void_p(stream.cuda_stream)
    lib = _lib.load()

    def step():
        _lib.check(lib.otf_pq_encode(local, _lib.tptr(x), n, dim, _lib.tptr(cents), M, K, Q, _lib.tptr(codes),
                                     _lib.MEM_DEVICE, sp))

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    steps = min(args.steps, 20)
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    launches0 = _lib.launch_count()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    with ClockSampler(local) as clk:
        for i in range(steps):
            starts[i].record(stream)
            step()
            ends[i].record(stream)
        torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    launches = _lib.launch_count() - launches0
    ms = float(np.mean([a.elapsed_time(b) for a, b in zip(starts, ends)]))
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = n * world / (ms / 1e3)
    flops = 2.0 * n * M * K * Q
    achieved = flops / (ms / 1e3) / 1e12

    # e2e through the public API: host vectors in, host codes out (a 1M-row batch per call)
    e2e_rows = min(n, 1_000_000)
    xh = x[:e2e_rows].cpu().numpy()
    book = otf.PQCodebook(cents_np)
    otf.pq_encode(book, xh[:1000])
    e2e_t = []
    for _ in range(3):
        t0 = time.perf_counter()
        otf.pq_encode(book, xh)
        e2e_t.append(time.perf_counter() - t0)
    e2e_s = float(np.mean(e2e_t))

    cpu = None
    if rank == 0 and not args.no_cpu:
        rows_c, fn, desc = cpu_sample(cfg)
        fn()
        t0 = time.perf_counter()
        fn()
        cpu = {"value": rows_c / (time.perf_counter() - t0), "unit": "vectors/s", "cores": cpu_threads(),
               "kind": "port", "sample": desc + ", oracle port (numpy, the reference's arithmetic), one run"}
    if rank == 0:
        metric, unit = metric_unit(cfg)
        line = {
            "metric": metric, "value": value, "unit": unit, "n_gpus": world, "steps": steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "tf32x3 / f32 screening, f64 decision", "data": "synthetic",
            "config": {"workload": cfg["workload"], "rows_per_gpu": n, "dim": dim, "blocks": M,
                       "centroids": K, "subdim": Q, "l2": "inputs (%.1f GB/GPU) larger than L2" % (n * dim * 4 / 1e9)},
            "roofline": {"bound": "fp32", "achieved": achieved, "peak": FP32_PEAK_TFLOPS, "unit": "TFLOP/s",
                         "frac": achieved / FP32_PEAK_TFLOPS, "traffic": profile_traffic("c3e"),
                         "traffic_unit": "DRAM bytes per launch (ncu)",
                         "kernel": ("pq_encode_mma: 2*K*Q useful flop per vector and block; the dots run as TF32x3 "
                                    "mma.sync tiles, the per-centroid distance + running argmin (SIMT ALU) bound it; "
                                    "peak = the FFMA form's bound"),
                         "hbm_gbs": n * (dim * 4 + M) / (ms / 1e3) / 1e9,
                         "peak_source": "derived: 148 SMs x 128 FFMA/clk x 2 x 1.965 GHz (no measured FP32 peak)"},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_rows / e2e_s, "unit": unit, "h2d_bytes_per_step": e2e_rows * dim * 4,
                    "d2h_bytes_per_step": e2e_rows * M, "rows_per_call": e2e_rows},
            "gpu_launches": launches,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def run_learn(args, cfg):
    """C3 codebook: learn_pq_codebook through the public API (host training matrix in, host
    codebook out — the call a user makes; every step's H2D/D2H is inside the timed region).
    GPU launches: the Lloyd assignment / objective / mean kernels of every block and iteration."""
    import torch

    import paper_1407_4764_b200 as otf
    from paper_1407_4764_b200 import _lib

    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    otf.set_device(local)
    rng = np.random.default_rng(1234)
    x = rng.standard_normal((cfg["rows"], cfg["dim"] * cfg["subdim"]), dtype=np.float32)
    x /= np.linalg.norm(x, axis=1, keepdims=True)
    pcfg = otf.PQConfig(subdim=cfg["subdim"], num_centroids=cfg["k"], iterations=cfg["iterations"], seed=5)
    for _ in range(args.warmup):
        otf.learn_pq_codebook(x, pcfg)
    steps = min(args.steps, 5)
    launches0 = _lib.launch_count()
    times = []
    with ClockSampler(local) as clk:
        for _ in range(steps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            book = otf.learn_pq_codebook(x, pcfg)
            times.append(time.perf_counter() - t0)
    launches = _lib.launch_count() - launches0
    ms = float(np.mean(times)) * 1e3
    iters = sum(len(h) for h in book.objective_history)
    n, K, Q = cfg["rows"], cfg["k"], cfg["subdim"]
    flops = 2.0 * n * K * Q * iters  # the assignment's float64 FMAs
    achieved = flops / (ms / 1e3) / 1e12
    cpu = None
    if rank == 0 and not args.no_cpu:
        scale, fn, desc = cpu_sample(cfg)
        t0 = time.perf_counter()
        fn()
        cpu = {"value": (time.perf_counter() - t0) * scale * 1e3, "unit": "ms", "cores": cpu_threads(), "kind": "port",
               "sample": desc + ", oracle port (numpy), one run"}
    if rank == 0:
        metric, unit = metric_unit(cfg)
        print(json.dumps({
            "metric": metric, "value": ms, "unit": unit, "n_gpus": 1, "steps": steps, "warmup": args.warmup,
            "ms_per_step": ms, "higher_is_better": False, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg["workload"], "rows": n, "blocks": cfg["dim"], "centroids": K, "subdim": Q,
                       "lloyd_iterations_run": iters, "l2": "training set (25.6 MB) is L2-resident by design"},
            "roofline": {"bound": "fp64", "achieved": achieved, "peak": 37.0, "unit": "TFLOP/s",
                         "frac": achieved / 37.0, "traffic": None,
                         "kernel": "km_assign (2*K*Q flop per training vector and iteration), whole call timed",
                         "peak_source": "nominal B200 FP64 (NVIDIA spec); the call is latency-bound "
                                        "(per-iteration host round trips), see DESIGN.md"},
            "cpu_baseline": cpu,
            "e2e": {"value": ms, "unit": unit, "h2d_bytes_per_step": n * cfg["dim"] * Q * 8,
                    "d2h_bytes_per_step": iters * (n * 4 + K * 8 + K * Q * 8 + 8)},
            "gpu_launches": launches // steps,
            "clocks": clk.summary(),
        }), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--train", dest="train", action="store_true", default=None,
                    help="run Pegasos steps concurrently with ranking (default: on for c4 only)")
    ap.add_argument("--no-train", dest="train", action="store_false")
    ap.add_argument("--group", choices=["torch", "native"], default="torch",
                    help="N>1 exchange: torch.distributed NCCL collectives (default) or the library's own "
                         "NCCL communicator (otf_group_*)")
    args = ap.parse_args()
    cfg = dict(CONFIGS[args.config])
    if os.environ.get("OTF_BENCH_ROWS"):  # profiling runs only: shrink the repository
        cfg["rows"] = int(os.environ["OTF_BENCH_ROWS"])
    if args.steps is None:
        args.steps = 20 if args.impl == "reference" else 500
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        return run_reference(args, cfg)
    if cfg["kind"] == "pqenc":
        return run_encode(args, cfg)
    if cfg["kind"] == "pqlearn":
        return run_learn(args, cfg)
    return run_gpu(args, cfg)


if __name__ == "__main__":
    sys.exit(main())
