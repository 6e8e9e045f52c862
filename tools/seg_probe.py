"""rank_many on a 64-classifier repository: fallbacks taken by the sampled-threshold selection
and its time against the histogram path (OTF_SEG_NO_CUT is read once per process: run twice)."""
import ctypes as C
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1407_4764_b200 as otf  # noqa: E402
from paper_1407_4764_b200 import _lib  # noqa: E402

n, d, c, k = int(sys.argv[1]), int(sys.argv[2]), 64, 1000
x = torch.randn(n, d, device="cuda")
x /= x.norm(dim=1, keepdim=True)
repo = otf.Repository.from_device("dense", x.data_ptr(), n, d)
W = np.random.default_rng(1).standard_normal((c, d))
models = [otf.LinearModel(w, 1, 1) for w in W]
for _ in range(2):
    repo.rank_many(models, k)
torch.cuda.synchronize()
t = []
for _ in range(5):
    t0 = time.perf_counter()
    repo.rank_many(models, k)
    t.append(time.perf_counter() - t0)
v = C.c_int64()
_lib.check(_lib.load().otf_repo_cut_fallbacks(repo.handle, C.byref(v)))
print(f"n {n} d {d}: rank_many {min(t) * 1e3:.2f} ms, fallbacks {v.value}")
