"""Error statistics of score_many against the exact float64 dot (for DESIGN.md)."""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_1407_4764_b200 as otf

rng = np.random.default_rng(3)
for n, d in [(20000, 4096), (20000, 512)]:
    x = rng.standard_normal((n, d)).astype(np.float32)
    x /= np.linalg.norm(x, axis=1, keepdims=True)
    W = rng.standard_normal((64, d))
    S = otf.Repository.dense(otf.FeatureStore(x)).score_many(list(W))
    ex = (x.astype(np.float64) @ W.astype(np.float32).astype(np.float64).T).T
    mag = np.abs(W.astype(np.float32).astype(np.float64)) @ np.abs(x.astype(np.float64)).T
    err = np.abs(S - ex)
    tol = 1e-6 * np.linalg.norm(W, axis=1)[:, None]
    f32 = np.abs((x @ W.astype(np.float32).T).T.astype(np.float64) - ex)  # numpy float32 sgemm
    print(f"d={d}: max err/mag = 2^{np.log2((err / mag).max()):.1f}, max err/(1e-6|w||x|) = {(err / tol).max():.3f}, "
          f"numpy f32 sgemm: max err/mag = 2^{np.log2((f32 / mag).max()):.1f}, err/tol {(f32 / tol).max():.3f}")
