"""How the C3 step (PQ scan + top-k) depends on k (the candidate count C grows with k)."""
import ctypes as C
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1407_4764_b200 as otf
from paper_1407_4764_b200 import _lib

n, m, q = 10_000_000, 16, 8
codes = torch.randint(0, 256, (n, m), dtype=torch.uint8, device="cuda")
cents = np.random.default_rng(1).standard_normal((m, 256, q)).astype(np.float32)
repo = otf.Repository.from_device("pq", codes.data_ptr(), n, m, codebook=otf.PQCodebook(cents))
w = torch.as_tensor(np.random.default_rng(2).standard_normal(m * q), device="cuda")
lib = _lib.load()
st = torch.cuda.current_stream()
for k in [1, 100, 300, 1000, 3000, 8000]:
    ids = torch.empty(k, dtype=torch.int64, device="cuda")
    sc = torch.empty(k, dtype=torch.float64, device="cuda")
    rows = torch.empty(k, dtype=torch.int64, device="cuda")
    call = lambda: _lib.check(lib.otf_repo_rank_graph(repo.handle, _lib.tptr(w), k, _lib.tptr(ids), _lib.tptr(sc),
                                                      _lib.tptr(rows), C.c_void_p(st.cuda_stream)))
    for _ in range(5):
        call()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(50):
        call()
    b.record()
    torch.cuda.synchronize()
    print(f"k={k}: {a.elapsed_time(b) / 50 * 1000:.1f} us per query")
