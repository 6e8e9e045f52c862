"""Error statistics of the dense and binary scans against the exact float64 dot and the
reference tolerance 1e-6 * ||w|| * ||x|| (for DESIGN.md), next to numpy's float32 sgemv."""
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "oracle")
import otf_oracle as O
import paper_1407_4764_b200 as otf

rng = np.random.default_rng(5)
for d in (128, 2048, 4096):
    x = rng.standard_normal((200_000, d)).astype(np.float32)
    x /= np.linalg.norm(x, axis=1, keepdims=True)
    w = rng.standard_normal(d)
    s = otf.Repository.dense(otf.FeatureStore(x)).score(w)
    ex = x.astype(np.float64) @ w.astype(np.float32).astype(np.float64)
    ref = O.score_dense(w, x)
    tol = 1e-6 * np.linalg.norm(w)
    print(f"dense d={d}: max |gpu-exact|/tol = {np.abs(s - ex).max() / tol:.4f}, "
          f"max |numpy-exact|/tol = {np.abs(ref - ex).max() / tol:.4f}, max |gpu-numpy|/tol = {np.abs(s - ref).max() / tol:.4f}")
bits = 2048
codes = rng.integers(0, 256, (200_000, bits // 8), dtype=np.uint8)
w = rng.standard_normal(bits)
s = otf.score_binary(w, codes, bits)
u = np.unpackbits(codes, axis=1, bitorder="little")[:, :bits].astype(np.float64)
ex = u @ w.astype(np.float32).astype(np.float64)
ref = O.score_binary(w, codes, bits)
tol = 1e-6 * np.linalg.norm(w) * np.sqrt(u.sum(1))
print(f"binary 2048: max |gpu-exact|/tol = {(np.abs(s - ex) / tol).max():.4f}, "
      f"max |numpy-exact|/tol = {(np.abs(ref - ex) / tol).max():.4f}")
