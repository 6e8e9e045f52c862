"""CPU oracle for the on-the-fly retrieval hot path — TEST INFRASTRUCTURE ONLY.

A numpy restatement of the reference's scoring / top-k / Pegasos arithmetic
(/root/reference/pkg/src/otf_retrieval, arXiv 1407.4764 reference package). Only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may import this
module, and only as the checker or the timed CPU baseline — the product path
(paper_1407_4764_b200) never calls it and has no CPU fallback.

Parity is pinned (tests/golden/): tests/golden/make_golden.py imports the real reference from
/root/reference in the build container, runs it on seeded inputs, and commits the outputs;
tests/test_oracle_golden.py checks this module against them bit-for-bit (integer/byte/PQ work)
or exactly-equal (dense/binary numpy calls are the same calls on the same host).

Besides the vectorised restatement, the two float64 reduction orders that make PQ scores
bit-exact are written out scalar-by-scalar (lut_entry_numpy_order, pairwise_sum_numpy_order):
these are the orders the CUDA kernels implement, and tests check them against numpy itself on
the machine the tests run on (the order is a property of the host numpy build).
"""

from __future__ import annotations

import math

import numpy as np

# ---------------------------------------------------------------------------------------------
# scoring — ranker.py:59-94, pq.py:248-276, binary.py:110-120


def as_weights(model) -> np.ndarray:
    """ranker.py:59-60: a LinearModel's weights or a bare array."""
    return np.asarray(getattr(model, "weights", model))


def score_dense(w, data) -> np.ndarray:
    """ranker.py:63-69: float32 matrix-vector product against float32(w)."""
    x = np.asarray(getattr(data, "data", data), dtype=np.float32)
    w = as_weights(w)
    if x.shape[1] != w.shape[0]:
        raise ValueError("dim mismatch")
    return x @ w.astype(np.float32)


def build_score_lut(w, centroids) -> np.ndarray:
    """pq.py:248-259: (M, K) float64 table of block inner products (full float64 w)."""
    cents = np.asarray(centroids, dtype=np.float32)
    m, _, q = cents.shape
    wb = np.asarray(w, dtype=np.float64).reshape(m, q)
    return np.einsum("mkq,mq->mk", cents.astype(np.float64), wb)


def score_codes(lut, codes, chunk_rows: int = 1 << 18) -> np.ndarray:
    """pq.py:262-276: one LUT read per block, float64 numpy (pairwise) sum per row."""
    arr = np.asarray(codes, dtype=np.uint8)
    out = np.empty(arr.shape[0], dtype=np.float64)
    cols = np.arange(lut.shape[0])
    for s in range(0, arr.shape[0], chunk_rows):
        e = min(s + chunk_rows, arr.shape[0])
        out[s:e] = lut[cols, arr[s:e]].sum(axis=1)
    return out


def score_pq(w, centroids, codes) -> np.ndarray:
    """ranker.py:72-75."""
    return score_codes(build_score_lut(w, centroids), codes)


def unpack_bits(codes, output_bits: int) -> np.ndarray:
    """binary.py:110-120: LSB-first bits as float32 {0, 1}, padding dropped."""
    arr = np.asarray(codes, dtype=np.uint8)
    return np.unpackbits(arr, axis=1, count=output_bits, bitorder="little").astype(np.float32)


def score_binary(w, codes, output_bits: int, chunk_rows: int = 1 << 14) -> np.ndarray:
    """ranker.py:78-94: unpack chunks to float32 {0,1} and sgemv with float32(w)."""
    arr = np.asarray(codes, dtype=np.uint8)
    w32 = as_weights(w).astype(np.float32)
    out = np.empty(arr.shape[0], dtype=np.float32)
    for s in range(0, arr.shape[0], chunk_rows):
        e = min(s + chunk_rows, arr.shape[0])
        out[s:e] = unpack_bits(arr[s:e], output_bits) @ w32
    return out


def hamming_distance(a, b) -> np.ndarray:
    """binary.py:123-128."""
    return np.bitwise_count(np.bitwise_xor(np.asarray(a, np.uint8), np.asarray(b, np.uint8))).sum(axis=-1).astype(np.int64)


def make_tight_frame(input_dim: int, output_bits: int, seed: int = 0) -> np.ndarray:
    """binary.py:46-66: first input_dim columns of the sign-pinned Q of a seeded Gaussian QR."""
    rng = np.random.default_rng(seed)
    q, r = np.linalg.qr(rng.standard_normal((output_bits, output_bits)))
    q = q * np.where(np.diag(r) < 0.0, -1.0, 1.0)[np.newaxis, :]
    return np.ascontiguousarray(q[:, :input_dim])


def binarize(frame: np.ndarray, centering, vectors) -> np.ndarray:
    """binary.py:86-107: bits of (x - mu) U^T > 0 in float64, packed LSB-first."""
    arr = np.atleast_2d(np.asarray(vectors, dtype=np.float64))
    proj = (arr - np.asarray(centering, dtype=np.float32).astype(np.float64)) @ frame.T
    return np.packbits(proj > 0.0, axis=1, bitorder="little")


# ---------------------------------------------------------------------------------------------
# explicit float64 orders (what the CUDA PQ kernels implement; pq.py:259 and pq.py:275)


def lut_entry_numpy_order(c, w) -> float:
    """One einsum('mkq,mq->mk') entry as numpy's SSE2 sum-of-products kernel computes it.

    Products are rounded separately (no FMA); two accumulators; each full 8-block adds
    p6,p4,p2,p0 into acc0 and p7,p5,p3,p1 into acc1; then remaining pairs (even->acc0,
    odd->acc1); a final odd element goes to acc0; result is 0.0 + (acc0 + acc1).
    """
    p = [float(a) * float(b) for a, b in zip(c, w)]
    q = len(p)
    acc0 = acc1 = 0.0
    i = 0
    while q - i >= 8:
        for j in (6, 4, 2, 0):
            acc0 += p[i + j]
            acc1 += p[i + j + 1]
        i += 8
    while q - i >= 2:
        acc0 += p[i]
        acc1 += p[i + 1]
        i += 2
    if i < q:
        acc0 += p[i]
    return 0.0 + (acc0 + acc1)


def pq_encode(centroids, vectors, chunk_rows: int = 1 << 18):
    """pq.py:206-230 — nearest centroid per sub-block in float64: argmin_j (|c_j|^2 - 2 x.c_j)
    (|x|^2 dropped), ties to the lowest index. Also returns the best and second-best distance
    of every (row, block), so a test can tell a genuine near-tie (|d1 - d2| at rounding level,
    where the BLAS dot order may pick either) from a real mismatch."""
    cents64 = np.asarray(centroids, dtype=np.float32).astype(np.float64)
    M, K, Q = cents64.shape
    arr = np.asarray(vectors, dtype=np.float32)
    norms = np.sum(cents64 * cents64, axis=2)
    n = arr.shape[0]
    codes = np.empty((n, M), dtype=np.uint8)
    gap = np.empty((n, M), dtype=np.float64)
    for start in range(0, n, chunk_rows):
        chunk = arr[start:start + chunk_rows].astype(np.float64)
        for m in range(M):
            sq = norms[m][np.newaxis, :] - 2.0 * (chunk[:, m * Q:(m + 1) * Q] @ cents64[m].T)
            a = np.argmin(sq, axis=1)
            codes[start:start + len(chunk), m] = a.astype(np.uint8)
            part = np.partition(sq, 1, axis=1) if K > 1 else np.concatenate([sq, sq + np.inf], axis=1)
            gap[start:start + len(chunk), m] = part[:, 1] - part[:, 0]
    return codes, gap


def lloyd(data, k: int, iterations: int, rng, init=None):
    """pq.py:100-171 — Lloyd k-means on one sub-block in float64: squared distances
    |x|^2 - 2 x.c + |c|^2, first-minimum assignment, objective = sum of clamped best distances
    (recorded before the update), stop when an assignment repeats after a plain update, means of
    non-empty clusters, each empty cluster re-seeded at the member of the (current) largest
    cluster farthest from its mean. Initial centroids: k distinct unique rows via rng.choice."""
    x = np.asarray(data, dtype=np.float64)
    if init is None:
        uniq = np.unique(x, axis=0)
        if uniq.shape[0] < k:
            raise ValueError("too few distinct rows")
        cents = uniq[rng.choice(uniq.shape[0], size=k, replace=False)].copy()
    else:
        cents = np.asarray(init, dtype=np.float64).copy()
    hist = []
    prev, plain = None, True
    for _ in range(iterations):
        d2 = (x * x).sum(1)[:, None] - 2.0 * (x @ cents.T) + (cents * cents).sum(1)[None, :]
        lab = d2.argmin(1)
        hist.append(float(np.maximum(d2[np.arange(len(x)), lab], 0.0).sum()))
        if prev is not None and plain and np.array_equal(lab, prev):
            break
        prev = lab
        cnt = np.bincount(lab, minlength=k)
        empty = np.flatnonzero(cnt == 0)
        plain = empty.size == 0
        for j in range(k):
            if cnt[j]:
                cents[j] = x[lab == j].mean(0)
        for j in empty:
            big = int(np.argmax(cnt))
            mem = np.flatnonzero(lab == big)
            far = mem[int(np.argmax(((x[mem] - cents[big]) ** 2).sum(1)))]
            cents[j] = x[far]
            lab[far] = j
            cnt[big] -= 1
            cnt[j] += 1
    return cents, hist


def learn_pq_codebook(train, subdim: int, k: int, iterations: int, seed: int):
    """pq.py:174-203 — blocks in order, one rng; returns (float32 centroids, histories, centering)."""
    data = np.asarray(train, dtype=np.float32)
    rng = np.random.default_rng(seed)
    blocks = data.shape[1] // subdim
    out = np.empty((blocks, k, subdim), dtype=np.float32)
    hists = []
    for m in range(blocks):
        c, h = lloyd(data[:, m * subdim:(m + 1) * subdim], k, iterations, rng)
        out[m] = c.astype(np.float32)
        hists.append(h)
    return out, hists, data.astype(np.float64).mean(0).astype(np.float32)


def pairwise_sum_numpy_order(a) -> float:
    """numpy's pairwise summation of a contiguous float64 run (add.reduce inner loop)."""
    n = len(a)
    if n < 8:
        res = -0.0
        for v in a:
            res += float(v)
        return res
    if n <= 128:
        r = [float(v) for v in a[:8]]
        i = 8
        while i < n - (n % 8):
            for j in range(8):
                r[j] += float(a[i + j])
            i += 8
        res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
        while i < n:
            res += float(a[i])
            i += 1
        return res
    n2 = n // 2
    n2 -= n2 % 8
    return pairwise_sum_numpy_order(a[:n2]) + pairwise_sum_numpy_order(a[n2:])


# ---------------------------------------------------------------------------------------------
# top-k — ranker.py:97-143


def top_k(scores, k: int, ids=None):
    """ranker.py:97-143: first k of the stable sort by (-score, id). Returns (ids, scores f64, rows)."""
    scores = np.asarray(scores)
    n = scores.shape[0]
    ids = np.arange(n, dtype=np.int64) if ids is None else np.asarray(ids, dtype=np.int64)
    k_eff = max(0, min(int(k), n))
    if k_eff == 0:
        return np.empty(0, np.int64), np.empty(0, np.float64), np.empty(0, np.int64)
    if k_eff == n:
        chosen = np.arange(n)
    else:
        thr = np.partition(scores, n - k_eff)[n - k_eff]
        above = np.flatnonzero(scores > thr)
        tie = np.flatnonzero(scores == thr)
        need = k_eff - above.size
        if need < tie.size:
            tie = tie[np.argsort(ids[tie], kind="stable")][:need]
        chosen = np.concatenate([above, tie])
    chosen = chosen[np.lexsort((ids[chosen], -scores[chosen].astype(np.float64)))]
    return ids[chosen].copy(), scores[chosen].astype(np.float64), chosen


def full_sort_ids(scores, ids, k):
    """The reference tests' independent oracle (tests/test_ranker.py:24-27)."""
    order = sorted(range(len(scores)), key=lambda i: (-float(scores[i]), int(ids[i])))
    return [int(ids[i]) for i in order[:k]]


# ---------------------------------------------------------------------------------------------
# Pegasos — trainer.py:51-106


def apply_update(w, t, batch, labels, lam, batch_size, project):
    """trainer.py:51-71."""
    eta = 1.0 / (lam * t)
    margins = labels * (batch @ w)
    viol = margins < 1.0
    grad = (labels[viol, np.newaxis] * batch[viol]).sum(axis=0)
    new_w = (1.0 - eta * lam) * w + (eta / batch_size) * grad
    if project:
        radius = 1.0 / math.sqrt(lam)
        norm = float(np.linalg.norm(new_w))
        if norm > radius:
            new_w *= radius / norm
    return new_w, viol


def pegasos_step(w, t, positives, negatives, lam, batch_size, project, rng, hook=None):
    """trainer.py:74-106 (validation elided): balanced draw, positives first."""
    half = batch_size // 2
    pi = rng.integers(0, len(positives), size=half)
    ni = rng.integers(0, len(negatives), size=half)
    if hook is not None:
        hook(pi, ni)
    batch = np.concatenate([np.asarray(positives, np.float64)[pi], np.asarray(negatives, np.float64)[ni]])
    labels = np.concatenate([np.ones(half), -np.ones(half)])
    new_w, _ = apply_update(np.asarray(w, np.float64), t, batch, labels, lam, batch_size, project)
    return new_w


def normalize_rows(data) -> np.ndarray:
    """store.py:32-53 (without the zero-norm check)."""
    arr = np.asarray(data, dtype=np.float64)
    return (arr / np.linalg.norm(arr, axis=1)[:, np.newaxis]).astype(np.float32)


def hinge_objective(w, features, labels, lam):
    """trainer.py:197-201."""
    w = np.asarray(w, dtype=np.float64)
    margins = labels * (np.asarray(features, dtype=np.float64) @ w)
    return float(0.5 * lam * np.dot(w, w) + np.maximum(0.0, 1.0 - margins).mean())


def train_batch(pos, neg, c=0.25, batch_size=32, epochs=60, project=True, seed=0, history=None):
    """trainer.py:204-257: Pegasos over the pooled set, tail average vs best epoch iterate."""
    feats = np.concatenate([np.asarray(pos, np.float64), np.asarray(neg, np.float64)])
    labels = np.concatenate([np.ones(len(pos)), -np.ones(len(neg))])
    n = len(feats)
    lam = 1.0 / (c * n)
    bs = min(batch_size, n)
    spe = math.ceil(n / bs)
    total = epochs * spe
    tail_len = max(1, total // 4)
    tail_start = total - tail_len
    rng = np.random.default_rng(seed)
    w = np.zeros(feats.shape[1])
    tail = np.zeros_like(w)
    best_obj, best_w = math.inf, w.copy()
    for t in range(1, total + 1):
        idx = rng.integers(0, n, size=bs)
        w, _ = apply_update(w, t, feats[idx], labels[idx], lam, bs, project)
        if t > tail_start:
            tail += w
        if t % spe == 0:
            obj = hinge_objective(w, feats, labels, lam)
            if history is not None:
                history.append(obj)
            if obj < best_obj:
                best_obj, best_w = obj, w.copy()
    avg = tail / tail_len
    return (avg if hinge_objective(avg, feats, labels, lam) <= best_obj else best_w), total


# ---------------------------------------------------------------------------------------------
# synthetic corpora — store.py:243-362 (the BASELINE.json C1 workload)


def generate_corpus_bundle(dim, classes, per_class, distractors, train_per_class, negative_count,
                           seed=0, cluster_spread=0.1, center_spread=1.0):
    """store.py:324-362: class centers, then train members (class by class), test members, the
    test distractors and the negative pool, all from ONE default_rng(seed) in that order, each
    store L2-normalised in float64 and cast to float32 (store.py:32-53). Returns
    (train (classes*train_per_class, dim), test (classes*per_class + distractors, dim),
    negatives (negative_count, dim)) float32; row r of a store has id r. Pinned by the CRC32s of
    the real reference's stores in tests/golden/golden_c1.npz."""
    rng = np.random.default_rng(seed)
    centers = rng.standard_normal((classes, dim)) * center_spread

    def members(n):
        return [centers[c] + rng.standard_normal((n, dim)) * cluster_spread for c in range(classes)]

    train = members(train_per_class)
    test = members(per_class)
    if distractors:
        test.append(rng.standard_normal((distractors, dim)) * center_spread)
    neg = rng.standard_normal((negative_count, dim)) * center_spread
    return normalize_rows(np.vstack(train)), normalize_rows(np.vstack(test)), normalize_rows(neg)
