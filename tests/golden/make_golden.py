"""Generate golden fixtures by running the REAL reference (build container only).

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Imports otf_retrieval from /root/reference/pkg/src (read-only), runs its hot-path functions on
seeded inputs and writes tests/golden/golden.npz. The GPU box has no /root/reference; the tests
only read the committed .npz. Inputs are stored next to outputs so nothing is regenerated.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent / "golden.npz"


def main() -> None:
    sys.path.insert(0, str(REF))
    sys.dont_write_bytecode = True
    from otf_retrieval import binary as rb
    from otf_retrieval import pq as rpq
    from otf_retrieval import ranker as rr
    from otf_retrieval import trainer as rt
    from otf_retrieval.model import LinearModel
    from otf_retrieval.store import FeatureStore, normalize_rows

    g: dict[str, np.ndarray] = {}

    # ---- dense scoring + ranking (ranker.py:63-69, :97-143, :272-281) --------------------
    for name, (n, d, seed) in {"d16": (200, 16, 3), "d128": (1500, 128, 5), "d2048": (120, 2048, 7),
                               "d5": (333, 5, 9)}.items():
        rng = np.random.default_rng(seed)
        x = normalize_rows(rng.standard_normal((n, d)))
        w = rng.standard_normal(d)
        ids = np.arange(n, dtype=np.int64) * 3 + 11
        rng.shuffle(ids)
        store = FeatureStore(x, ids=ids)
        repo = rr.Repository.dense(store)
        ranked = repo.rank(LinearModel(w, 1, 4), 50)
        g[f"dense_{name}_x"] = x
        g[f"dense_{name}_w"] = w
        g[f"dense_{name}_ids"] = ids
        g[f"dense_{name}_scores"] = repo.score(w)
        g[f"dense_{name}_rank_ids"] = ranked.ids
        g[f"dense_{name}_rank_scores"] = ranked.scores

    # ---- PQ (pq.py:248-276) — bit-exact targets ------------------------------------------
    for name, (m, k, q, n, seed) in {"m4k8q4": (4, 8, 4, 500, 11), "m16k256q8": (16, 256, 8, 3000, 12),
                                     "m5k7q3": (5, 7, 3, 300, 13), "m32k256q4": (32, 256, 4, 2000, 14),
                                     "m12k200q16": (12, 200, 16, 600, 15), "m200k16q1": (200, 16, 1, 300, 16)}.items():
        rng = np.random.default_rng(seed)
        cents = (rng.standard_normal((m, k, q)) * np.exp(rng.uniform(-3, 3, size=(m, k, 1)))).astype(np.float32)
        book = rpq.PQCodebook(cents, np.zeros(m * q, dtype=np.float32))
        codes = rng.integers(0, k, size=(n, m)).astype(np.uint8)
        w = rng.standard_normal(m * q) * np.exp(rng.uniform(-2, 2, size=m * q))
        lut = rpq.build_score_lut(w, book)
        repo = rr.Repository.quantized(book, codes)
        ranked = repo.rank(LinearModel(w, 1, 1), 40)
        g[f"pq_{name}_cents"] = cents
        g[f"pq_{name}_codes"] = codes
        g[f"pq_{name}_w"] = w
        g[f"pq_{name}_lut"] = lut
        g[f"pq_{name}_scores"] = rpq.score_codes(lut, codes)
        g[f"pq_{name}_rank_ids"] = ranked.ids
        g[f"pq_{name}_rank_scores"] = ranked.scores

    # ---- pq_encode (pq.py:206-230): codes of fresh vectors under a learned codebook ------------
    for name, (m, k, q, n_train, n, seed) in {"e16": (16, 256, 8, 3000, 2000, 61),
                                              "e4k16": (4, 16, 5, 400, 700, 62)}.items():
        rng = np.random.default_rng(seed)
        train = normalize_rows(rng.standard_normal((n_train, m * q))).astype(np.float32)
        book = rpq.learn_pq_codebook(train, rpq.PQConfig(subdim=q, num_centroids=k, iterations=6, seed=seed))
        vecs = normalize_rows(rng.standard_normal((n, m * q))).astype(np.float32)
        vecs[:5] = book.centroids[:, :5, :].transpose(1, 0, 2).reshape(5, m * q)  # exact centroid hits
        g[f"pqenc_{name}_cents"] = book.centroids
        g[f"pqenc_{name}_vecs"] = vecs
        g[f"pqenc_{name}_codes"] = rpq.pq_encode(book, vecs)

    # ---- codebook learning (pq.py:116-203): learn_pq_codebook and _lloyd traces ----------------
    for name, (n, d, q, k, iters, seed) in {"a": (3000, 16, 8, 64, 10, 3), "b": (1200, 12, 3, 16, 25, 4)}.items():
        rng = np.random.default_rng(seed)
        train = normalize_rows(rng.standard_normal((n, d))).astype(np.float32)
        book = rpq.learn_pq_codebook(train, rpq.PQConfig(subdim=q, num_centroids=k, iterations=iters, seed=seed))
        hist = book.objective_history
        width = max(len(h) for h in hist)
        g[f"km_{name}_train"] = train
        g[f"km_{name}_cents"] = book.centroids
        g[f"km_{name}_centering"] = book.centering
        g[f"km_{name}_hist"] = np.array([h + [np.nan] * (width - len(h)) for h in hist])
        g[f"km_{name}_hist_len"] = np.array([len(h) for h in hist])
    hand_c, hand_h = rpq._lloyd(np.array([[0.0], [1.0], [2.0], [3.0]]), k=2, iterations=10,
                                rng=np.random.default_rng(0), init=np.array([[0.0], [1000.0]]))
    g["km_hand_cents"], g["km_hand_hist"] = hand_c, np.array(hand_h)
    rng = np.random.default_rng(77)
    data = rng.standard_normal((400, 3))
    init = np.concatenate([data[:5], np.full((3, 3), 50.0)])  # three far centroids -> empty clusters
    emp_c, emp_h = rpq._lloyd(data, k=8, iterations=15, rng=np.random.default_rng(1), init=init)
    g["km_empty_data"], g["km_empty_init"] = data, init
    g["km_empty_cents"], g["km_empty_hist"] = emp_c, np.array(emp_h)

    # ---- binary (ranker.py:78-94, binary.py:86-128) ----------------------------------------
    for name, (m, bits, n, seed) in {"b32": (8, 32, 200, 21), "b2048": (128, 2048, 300, 22),
                                     "b19": (8, 19, 150, 23), "b1024": (64, 1024, 300, 24)}.items():
        rng = np.random.default_rng(seed)
        frame = rb.make_tight_frame(m, bits, seed=seed)
        codec = rb.BinaryCodec(frame, rng.standard_normal(m).astype(np.float32) * 0.1)
        vecs = rng.standard_normal((n, m))
        codes = rb.binarize(codec, vecs)
        w = rng.standard_normal(bits)
        repo = rr.Repository.binary(codec, codes)
        ranked = repo.rank(LinearModel(w, 1, 2), 30)
        if bits <= 1024:  # the 2048-bit frame (2 MB) is not needed to check scoring
            g[f"bin_{name}_frame"] = frame.matrix
            g[f"bin_{name}_center"] = codec.centering
            g[f"bin_{name}_vecs"] = vecs
        g[f"bin_{name}_codes"] = codes
        g[f"bin_{name}_w"] = w
        g[f"bin_{name}_scores"] = rr.score_binary(w, codes, bits)
        g[f"bin_{name}_unpacked"] = rb.unpack_bits(codes[:20], bits)
        g[f"bin_{name}_rank_ids"] = ranked.ids
        g[f"bin_{name}_rank_scores"] = ranked.scores
        other = rng.integers(0, 256, size=codes.shape).astype(np.uint8)
        g[f"bin_{name}_other"] = other
        g[f"bin_{name}_hamming"] = rb.hamming_distance(codes, other)
        g[f"bin_{name}_adapted"] = repo.adapt_training_vectors(vecs[:10])

    # ---- top_k known answers + ties (tests/test_ranker.py:139-197) -------------------------
    rng = np.random.default_rng(11)
    ties = rng.integers(0, 5, size=10_000).astype(np.float32)
    tie_ids = np.arange(10_000, dtype=np.int64)
    rng.shuffle(tie_ids)
    r = rr.top_k(ties, 100, ids=tie_ids)
    g["topk_ties_scores"], g["topk_ties_ids_in"] = ties, tie_ids
    g["topk_ties_ids"], g["topk_ties_out_scores"] = r.ids, r.scores
    rnd = np.random.default_rng(12).standard_normal(5000).astype(np.float32)
    r = rr.top_k(rnd, 50)
    g["topk_rand_scores"], g["topk_rand_ids"] = rnd, r.ids
    sgn = np.array([0.0, -0.0, 1.0, -0.0, 0.0, -1.0], dtype=np.float32)
    r = rr.top_k(sgn, 4)
    g["topk_signed_zero_scores"], g["topk_signed_zero_ids"] = sgn, r.ids
    f64 = np.random.default_rng(13).integers(-3, 4, size=3000).astype(np.float64) / 7.0
    r = rr.top_k(f64, 1000)
    g["topk_f64_scores"], g["topk_f64_ids"] = f64, r.ids
    r = rr.top_k(f64[:700], 5000)
    g["topk_full_ids"] = r.ids

    # ---- Pegasos (trainer.py:51-173) ---------------------------------------------------------
    rng = np.random.default_rng(31)
    d = 24
    pos = normalize_rows(rng.standard_normal((40, d)) + 1.5)
    neg = normalize_rows(rng.standard_normal((300, d)) - 0.5)
    batches: list[np.ndarray] = []
    tr = rt.OnlineTrainer(d, neg, rt.TrainerConfig(lam=0.05, batch_size=16, seed=9),
                          batch_hook=lambda p, q: batches.append(np.concatenate([p, q])))
    ws = []
    for _ in range(60):
        tr.step(pos)
        ws.append(tr.snapshot().weights)
    g["peg_pos"], g["peg_neg"] = pos, neg
    g["peg_idx"] = np.stack(batches)
    g["peg_w"] = np.stack(ws)
    # stateless pegasos_step sequence with project=False and float64 pools
    rng2 = np.random.default_rng(5)
    w = np.zeros(d)
    seq = []
    cfg = rt.TrainerConfig(lam=0.3, batch_size=8, project=False, seed=0)
    for t in range(1, 31):
        w = rt.pegasos_step(w, t, pos.astype(np.float64), neg.astype(np.float64), cfg, rng2)
        seq.append(w)
    g["peg_noproj_w"] = np.stack(seq)

    # ---- fixed-set SVM (trainer.py:197-257) ---------------------------------------------------
    for name, (n_pos, n_neg, d, epochs, seed) in {"tb16": (60, 400, 16, 20, 41), "tb128": (40, 600, 128, 8, 42)}.items():
        rng = np.random.default_rng(seed)
        pos = normalize_rows(rng.standard_normal((n_pos, d)) + 0.8)
        neg = normalize_rows(rng.standard_normal((n_neg, d)))
        hist: list[float] = []
        model = rt.train_batch(pos, neg, rt.BatchTrainConfig(c=0.25, epochs=epochs, seed=seed), objective_history=hist)
        feats = np.concatenate([pos, neg]).astype(np.float64)
        labels = np.concatenate([np.ones(n_pos), -np.ones(n_neg)])
        g[f"tb_{name}_pos"], g[f"tb_{name}_neg"] = pos, neg
        g[f"tb_{name}_w"] = model.weights
        g[f"tb_{name}_iter"] = np.array([model.iteration])
        g[f"tb_{name}_hist"] = np.array(hist)
        g[f"tb_{name}_obj"] = np.array([rt.hinge_objective(model.weights, feats, labels, 1.0 / (0.25 * len(feats)))])

    # ---- live session replay (session.py:237-290) ---------------------------------------------
    from otf_retrieval import session as rs
    from otf_retrieval.store import SynthConfig, generate_corpus_bundle

    bundle = generate_corpus_bundle(SynthConfig(dim=32, classes=3, per_class=40, distractors=3000, seed=51),
                                    train_per_class=30, negative_count=400)
    repo = rr.Repository.dense(bundle.test)
    cfg = rs.SessionConfig(rate=12.0, ranker=rr.RankerConfig(k=25, interval=0.18),
                           trainer=rt.TrainerConfig(lam=0.1, batch_size=16), steps_per_second=100.0)
    sess = rs.QuerySession("s", "class_00", repo, bundle.negatives.data, cfg, trainer_seed=5)
    train_rows = sorted(bundle.train_labels.ids_for("class_00"))
    feed = bundle.train.data[train_rows]
    pubs = []
    rs.run_simulated(sess, feed, 2.0, on_publish=pubs.append)
    g["sess_test_x"], g["sess_neg"], g["sess_feed"] = bundle.test.data, bundle.negatives.data, feed
    g["sess_ids"] = np.stack([p.ranked.ids for p in pubs])
    g["sess_meta"] = np.array([[p.ranked.model_version, p.positives_fed, p.steps_applied, p.lists_published]
                               for p in pubs])
    g["sess_at"] = np.array([p.ranked.produced_at for p in pubs])
    g["sess_w"] = sess.trainer.snapshot().weights

    np.savez_compressed(OUT, **g)
    print(f"wrote {OUT} ({OUT.stat().st_size} bytes, {len(g)} arrays)")


if __name__ == "__main__":
    main()
