"""Where the end-to-end query time goes (host w in -> host RankedList out), per config:
  api     Repository.rank(model, k)                      (Python + ctypes + C host path)
  ctypes  lib.otf_repo_rank(... MEM_HOST ...) with prepared arguments (C host path)
  device  otf_repo_rank_graph on device buffers + stream sync (graph replay, no copies)
  events  the same replay timed with CUDA events (GPU time only)
    python tools/latency_probe.py c1 c3
"""

import ctypes as C
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1407_4764_b200 as otf  # noqa: E402
from paper_1407_4764_b200 import _lib  # noqa: E402


def stats(ts):
    ts = np.sort(np.asarray(ts) * 1e6)
    return f"median {np.median(ts):7.1f} us  p10 {ts[len(ts) // 10]:7.1f}  p90 {ts[9 * len(ts) // 10]:7.1f}"


def probe(name):
    cfg = dict(bench.CONFIGS[name])
    repo, keep, _ = bench.make_repository(cfg, 0, 1, 0)
    dim = repo.model_dim
    k = cfg["k"]
    w = bench.query_weights(cfg, dim)
    model = otf.LinearModel(w, 1, 1)
    lib = _lib.load()
    reps = 300
    for _ in range(20):
        repo.rank(model, k)
    api = []
    for _ in range(reps):
        t0 = time.perf_counter()
        repo.rank(model, k)
        api.append(time.perf_counter() - t0)
    ids = np.empty(k, np.int64)
    sc = np.empty(k, np.float64)
    got = C.c_int64()
    args = (repo.handle, _lib.ptr(np.ascontiguousarray(w)), k, _lib.ptr(ids), _lib.ptr(sc), None, C.byref(got),
            _lib.MEM_HOST, None)
    cty = []
    for _ in range(reps):
        t0 = time.perf_counter()
        lib.otf_repo_rank(*args)
        cty.append(time.perf_counter() - t0)
    dev = torch.device("cuda", 0)
    w_dev = torch.as_tensor(w, device=dev)
    o_ids = torch.empty(k, dtype=torch.int64, device=dev)
    o_sc = torch.empty(k, dtype=torch.float64, device=dev)
    o_rows = torch.empty(k, dtype=torch.int64, device=dev)
    st = torch.cuda.current_stream(dev)
    sp = C.c_void_p(st.cuda_stream)
    gr = []
    for _ in range(reps):
        t0 = time.perf_counter()
        lib.otf_repo_rank_graph(repo.handle, _lib.tptr(w_dev), k, _lib.tptr(o_ids), _lib.tptr(o_sc), _lib.tptr(o_rows),
                                sp)
        st.synchronize()
        gr.append(time.perf_counter() - t0)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev = []
    for _ in range(reps):
        e0.record(st)
        lib.otf_repo_rank_graph(repo.handle, _lib.tptr(w_dev), k, _lib.tptr(o_ids), _lib.tptr(o_sc), _lib.tptr(o_rows),
                                sp)
        e1.record(st)
        st.synchronize()
        ev.append(e0.elapsed_time(e1) * 1e-3)
    print(f"{name}: api    {stats(api)}")
    print(f"{name}: ctypes {stats(cty)}")
    print(f"{name}: device {stats(gr)}")
    print(f"{name}: events {stats(ev)}", flush=True)
    del repo, keep


if __name__ == "__main__":
    for name in sys.argv[1:] or ["c1", "c3"]:
        probe(name)
