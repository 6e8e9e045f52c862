"""Repository.score on a 10M x 16 PQ repository (float64 scores): event-timed, with a digest of the
scores so two runs (default pq_score16_lines; OTF_PQ_SCORE_XOR=1 for pq_scan16_xor) can be compared."""
import hashlib
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import ctypes as C  # noqa: E402

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1407_4764_b200 as otf  # noqa: E402
from paper_1407_4764_b200 import _lib  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
rng = np.random.default_rng(1)
cents = rng.standard_normal((16, 256, 8)).astype(np.float32)
torch.manual_seed(1)
codes = torch.randint(0, 256, (n, 16), dtype=torch.uint8, device="cuda")
repo = otf.Repository.from_device("pq", codes.data_ptr(), n, 16, codebook=otf.PQCodebook(cents))
w = torch.as_tensor(rng.standard_normal(128), device="cuda")
out = torch.empty(n, dtype=torch.float64, device="cuda")
lib = _lib.load()
st = torch.cuda.current_stream()
sp = C.c_void_p(st.cuda_stream)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ts = []
for i in range(30):
    e0.record(st)
    _lib.check(lib.otf_repo_score(repo.handle, _lib.tptr(w), _lib.tptr(out), _lib.MEM_DEVICE, sp))
    e1.record(st)
    st.synchronize()
    if i >= 5:
        ts.append(e0.elapsed_time(e1) * 1e3)
t = float(np.median(ts))
print(f"score n={n}: {t:.1f} us (LUT + scan), {(n * 16 + n * 8) / t / 1e3:.2f} GB/s of codes + scores")
print("digest", hashlib.sha1(out.cpu().numpy().tobytes()).hexdigest())
