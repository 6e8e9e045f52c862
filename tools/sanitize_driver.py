"""Small workloads that launch every kernel family once, for compute-sanitizer runs
(tools/gpu_sanitize.sh): memcheck, racecheck (shared-memory hazards), synccheck (barrier misuse).
Each case also checks its result against the oracle so a silent corruption would fail here too."""

import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))

import numpy as np  # noqa: E402

import otf_oracle as O  # noqa: E402
import paper_1407_4764_b200 as otf  # noqa: E402

which = set(sys.argv[1:]) or {"dense", "pq", "pqcut", "binary", "multi", "train", "encode", "kmeans", "topk"}
rng = np.random.default_rng(0)

if "dense" in which:  # dense_score_fast + topk_coop_kernel (grid barrier, chunk maxima)
    x = rng.standard_normal((200_000, 128)).astype(np.float32)
    w = rng.standard_normal(128)
    repo = otf.Repository.dense(otf.FeatureStore(x))
    s = repo.score(w)
    r = repo.rank(otf.LinearModel(w, 1, 1), 500)
    ids, _, _ = O.top_k(s, 500)
    assert list(r.ids) == list(ids)
    print("dense ok")

if "topk" in which:  # radix-select path: heavy ties (w = 0)
    x = rng.standard_normal((50_000, 64)).astype(np.float32)
    repo = otf.Repository.dense(otf.FeatureStore(x))
    r = repo.rank(otf.LinearModel(np.zeros(64), 1, 1), 300)
    assert list(r.ids) == list(range(300))
    print("topk radix ok")

if "pq" in which:  # pq_build_lut_kernel + pq_scan16_f32bins + topk PqBinSrc; pq_scan16_xor (score)
    cents = rng.standard_normal((16, 256, 8)).astype(np.float32)
    codes = rng.integers(0, 256, (300_000, 16), dtype=np.uint8)
    w = rng.standard_normal(128)
    repo = otf.Repository.quantized(otf.PQCodebook(cents), codes)
    ref = O.score_pq(w, cents, codes)
    assert repo.score(w).tobytes() == ref.tobytes()
    r = repo.rank(otf.LinearModel(w, 1, 1), 200)
    assert list(r.ids) == list(O.top_k(ref, 200)[0])
    print("pq bins ok")

if "pqcut" in which:  # pq_rank_cut_kernel (TMA ring, mbarriers, grid barriers, emission, selection)
    cents = rng.standard_normal((16, 256, 8)).astype(np.float32)
    codes = rng.integers(0, 256, (3_000_000, 16), dtype=np.uint8)
    w = rng.standard_normal(128)
    repo = otf.Repository.quantized(otf.PQCodebook(cents), codes)
    ref = O.score_pq(w, cents, codes)
    r = repo.rank(otf.LinearModel(w, 1, 1), 100)
    assert list(r.ids) == list(O.top_k(ref, 100)[0])
    print("pq cut ok")

if "binary" in which:  # bin_score_bytes (2 slices) + topk
    codes = rng.integers(0, 256, (100_000, 256), dtype=np.uint8)
    w = rng.standard_normal(2048)
    s = otf.score_binary(w, codes, 2048)
    assert np.max(np.abs(s.astype(np.float64) - O.score_binary(w, codes, 2048))) < 1e-3
    print("binary ok")

if "multi" in which:  # multi_score_tc (tcgen05, TMA, TMEM, CTA pairs) + segmented top-k
    x = rng.standard_normal((20_000, 512)).astype(np.float32)
    W = rng.standard_normal((64, 512))
    repo = otf.Repository.dense(otf.FeatureStore(x))
    S = repo.score_many(list(W))
    for c in (0, 63):
        assert np.max(np.abs(S[c].astype(np.float64) - O.score_dense(W[c], x))) < 1e-3
    lists = repo.rank_many([otf.LinearModel(wc, 1, 1) for wc in W], 50)
    assert list(lists[5].ids) == list(O.top_k(S[5], 50)[0])
    print("multi ok")

if "train" in which:  # pegasos_kernel, batch_train_kernel, hinge objective
    neg = rng.standard_normal((500, 32)).astype(np.float32)
    pos = (rng.standard_normal((40, 32)) + 1.0).astype(np.float32)
    tr = otf.OnlineTrainer(32, neg, otf.TrainerConfig(lam=0.1, batch_size=8, seed=1))
    for _ in range(5):
        tr.step(pos)
    m = otf.train_batch(pos, neg, otf.BatchTrainConfig(c=0.25, epochs=2))
    assert np.all(np.isfinite(m.weights))
    print("train ok")

if "encode" in which:  # pq_encode_mma
    cents = rng.standard_normal((16, 256, 8)).astype(np.float32)
    x = rng.standard_normal((5_000, 128)).astype(np.float32)
    enc = otf.pq_encode(otf.PQCodebook(cents), x)
    ref, gap = O.pq_encode(cents, x)
    assert np.all((enc == ref) | (gap <= 1e-9))
    print("encode ok")

if "kmeans" in which:  # km_assign / objective / means
    x = rng.standard_normal((3_000, 32)).astype(np.float32)
    book = otf.learn_pq_codebook(x, otf.PQConfig(subdim=8, num_centroids=16, iterations=3, seed=1))
    assert np.all(np.isfinite(book.centroids))
    print("kmeans ok")
print("sanitize driver done")
