"""Randomised sweep of the fused selections (dense_rank_cut, pq_rank_cut_kernel,
topk_seg_cut_kernel) at the sizes where they run: every list must equal the oracle's top_k
(ranker.py:97-143) of the GPU's own scores (PQ: of the reference's bit-identical scores), for
continuous / tie-heavy / constant data, shuffled or negative ids, k from 1 to the plans' caps.
Prints one line per failure and the number of fallbacks taken. Run on a GPU box:
    python tools/stress_cut.py [cases_per_kind]
"""
import ctypes as C
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))

import numpy as np  # noqa: E402

import otf_oracle as O  # noqa: E402
import paper_1407_4764_b200 as otf  # noqa: E402
from paper_1407_4764_b200 import _lib  # noqa: E402


def fallbacks(repo):
    v = C.c_int64()
    _lib.check(_lib.load().otf_repo_cut_fallbacks(repo.handle, C.byref(v)))
    return v.value


class Store:
    def __init__(self, data, ids):
        self.data, self.ids = data, ids


def check(repo, w, k, ids, s=None):
    r = repo.rank(otf.LinearModel(w, 1, 1), k)
    if s is None:
        s = repo.score(w)
    o_ids, o_sc, _ = O.top_k(s, k, ids)
    if not np.array_equal(r.ids, o_ids) or r.scores.tobytes() != np.asarray(o_sc, np.float64).tobytes():
        return False
    return True


def main():
    cases = int(sys.argv[1]) if len(sys.argv) > 1 else 40
    bad = fb = 0
    t0 = time.time()
    for seed in range(cases):  # dense
        rng = np.random.default_rng(7000 + seed)
        d = int(rng.choice([128, 256, 512, 2048]))
        n = int(rng.integers(160_000, 3_000_000 if d <= 256 else 400_000))
        k = int(rng.choice([1, 10, 100, 1000, 1216]))
        dist = rng.choice(["cont", "cont", "ties", "const"])
        x = rng.standard_normal((n, d), dtype=np.float32)
        if dist == "ties":
            x = np.round(x * 2) / 2
        elif dist == "const":
            x[:] = 0.25
        ids = None if rng.random() < 0.5 else (rng.permutation(2 * n)[:n].astype(np.int64) - n)
        repo = otf.Repository.dense(Store(x, ids) if ids is not None else x)
        w = rng.standard_normal(d)
        ok = check(repo, w, k, ids)
        fb += fallbacks(repo)
        if not ok:
            bad += 1
            print(f"FAIL dense seed {seed} n {n} d {d} k {k} {dist}", flush=True)
        del repo, x
    print(f"dense done {time.time() - t0:.0f}s failures {bad} fallbacks {fb}", flush=True)
    for seed in range(cases // 2):  # PQ, M = 16
        rng = np.random.default_rng(8000 + seed)
        n = int(rng.integers(2_500_000, 12_000_000))
        k = int(rng.choice([1, 10, 100, 1000, 1100]))
        dist = rng.choice(["cont", "cont", "ties", "const"])
        cents = rng.standard_normal((16, 256, 8)).astype(np.float32)
        if dist == "ties":
            cents = np.round(cents)
        elif dist == "const":
            cents[:] = 0.5
        codes = rng.integers(0, 256, (n, 16), dtype=np.uint8)
        ids = None if rng.random() < 0.5 else (rng.permutation(2 * n)[:n].astype(np.int64) - n)
        repo = otf.Repository.quantized(otf.PQCodebook(cents), codes, ids=ids)
        w = rng.standard_normal(128)
        ok = check(repo, w, k, ids, O.score_pq(w, cents, codes))
        fb += fallbacks(repo)
        if not ok:
            bad += 1
            print(f"FAIL pq seed {seed} n {n} k {k} {dist}", flush=True)
        del repo, codes
    print(f"pq done {time.time() - t0:.0f}s failures {bad} fallbacks {fb}", flush=True)
    for seed in range(max(2, cases // 8)):  # many classifiers
        rng = np.random.default_rng(9000 + seed)
        n = int(rng.integers(1_048_576, 2_500_000))
        c = int(rng.choice([3, 17, 64]))
        k = int(rng.choice([1, 100, 1000]))
        x = np.round(rng.standard_normal((n, 64)) * 8).astype(np.float32) / 8
        W = rng.standard_normal((c, 64))
        W[0] = 0.0
        repo = otf.Repository.dense(x)
        S = repo.score_many(list(W))
        lists = repo.rank_many([otf.LinearModel(wc, 1, 1) for wc in W], k)
        for i in range(c):
            o_ids, o_sc, _ = O.top_k(S[i], k)
            if not np.array_equal(lists[i].ids, o_ids) or not np.array_equal(lists[i].scores, o_sc):
                bad += 1
                print(f"FAIL many seed {seed} n {n} c {c} k {k} classifier {i}", flush=True)
                break
        fb += fallbacks(repo)
        del repo, x
    print(f"stress_cut done {time.time() - t0:.0f}s, failures: {bad}, fallbacks taken: {fb}", flush=True)


if __name__ == "__main__":
    main()
