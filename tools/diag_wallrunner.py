"""Diagnose WallRunner progress under a busy-polling reader (GPU box)."""
import sys, time, threading
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import paper_1407_4764_b200 as otf
from paper_1407_4764_b200 import session as S

def clusters(dim, n_pos, n_neg, seed):
    rng = np.random.default_rng(seed)
    c = rng.standard_normal(dim)
    pos = (c + 0.3 * rng.standard_normal((n_pos, dim))).astype(np.float32)
    neg = rng.standard_normal((n_neg, dim)).astype(np.float32)
    return pos / np.linalg.norm(pos, axis=1, keepdims=True), neg / np.linalg.norm(neg, axis=1, keepdims=True)

for hog in (False, True, True):
    pos, neg = clusters(16, 400, 150, 8)
    x = np.random.default_rng(3).standard_normal((20_000, 16)).astype(np.float32)
    repo = otf.Repository.dense(otf.FeatureStore(x))
    cfg = S.SessionConfig(rate=200.0, ranker=otf.RankerConfig(k=25, interval=0.01),
                          trainer=otf.TrainerConfig(lam=0.02, batch_size=16), steps_per_second=500.0)
    sess = S.QuerySession("s", "q", repo, neg, cfg, trainer_seed=5)
    orig = sess.rank_tick
    ticks = []
    def tick(now):
        t0 = time.perf_counter(); r = orig(now); ticks.append((time.perf_counter() - t0, r)); return r
    sess.rank_tick = tick
    runner = S.WallRunner(sess, pos)
    t0 = time.monotonic()
    runner.start()
    polls = 0
    first = None
    while time.monotonic() < t0 + 0.8:
        if hog:
            p = sess.latest_publication(); polls += 1
            if p is not None and first is None: first = time.monotonic() - t0
        else:
            time.sleep(0.001)
            if first is None and sess.latest_publication() is not None: first = time.monotonic() - t0
    runner.stop()
    print(f"hog={hog} polls={polls} stats={sess.stats()} errors={runner.errors} first_pub_at={first} "
          f"ticks={len(ticks)} tick_ms={[round(a*1e3,2) for a,_ in ticks[:8]]} ok={[r for _,r in ticks[:8]]}", flush=True)
