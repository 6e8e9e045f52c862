"""GPU parity: the sm_100a path (through the C ABI) against the reference's own outputs
(tests/golden, produced by the unmodified reference) and against the pinned oracle.

Bars:
  * PQ: LUT, scores, ranked ids and ranked scores bit-identical.
  * top_k given the same scores: ids bit-identical (all edge cases of tests/test_ranker.py).
  * dense / binary scores: |gpu - ref| <= 1e-6 * ||w||_2 * ||x||_2 (the reference's own sgemv
    order is host-dependent); dense scores also stay within the kernel's documented bound
    (4-term float32 FMA chains summed in float64), binary scores within half an ulp.
  * ranked ids: identical to the oracle's top_k of the GPU's own scores (selection is exact) and
    equal as sets / in order to the reference up to swaps of entries whose reference scores are
    within that tolerance.
  * Pegasos: w within rtol 1e-12 of the reference at every step, same sampled indices.
"""

import numpy as np
import pytest

import otf_oracle as O

pytestmark = pytest.mark.gpu

DENSE = ["d16", "d128", "d2048", "d5"]
PQ = ["m4k8q4", "m16k256q8", "m5k7q3", "m32k256q4", "m12k200q16", "m200k16q1"]
BIN = ["b32", "b2048", "b19", "b1024"]


def assert_rank_parity(got_ids, ref_ids, ref_score_of, tol):
    """Set equality and order equality up to swaps of near-tied (|ds| <= tol) entries."""
    got_ids, ref_ids = list(map(int, got_ids)), list(map(int, ref_ids))
    assert len(got_ids) == len(ref_ids)
    if got_ids == ref_ids:
        return 0
    # allow boundary differences only between near-ties with the last reference entry
    last = ref_score_of[ref_ids[-1]]
    extra = set(got_ids) ^ set(ref_ids)
    for i in extra:
        assert abs(ref_score_of[i] - last) <= tol, f"id {i} differs beyond tolerance"
    swaps = 0
    for a, b in zip(got_ids, ref_ids):
        if a != b:
            swaps += 1
            if a in ref_score_of and b in ref_score_of:
                assert abs(ref_score_of[a] - ref_score_of[b]) <= tol
    return swaps


def exact_dense(x, w):
    return x.astype(np.float64) @ w.astype(np.float32).astype(np.float64)


def dense_error_bound(s, x, w):
    """Half an ulp of the float32 result plus the rounding of the 4-term float32 FMA chains
    (2^-22 * sum |x_j w_j|, generous) — the kernel's documented arithmetic (otf_dense.cu)."""
    mag = np.abs(x.astype(np.float64)) @ np.abs(w.astype(np.float32).astype(np.float64))
    return np.spacing(np.abs(s)) * 0.5 + 2.0 ** -22 * mag + 1e-30


# ---------------------------------------------------------------------------------------------
# dense (ranker.py:63-69, :272-281)


@pytest.mark.parametrize("name", DENSE)
def test_dense_scores_and_rank(otf, golden, name):
    x, w, ids = golden[f"dense_{name}_x"], golden[f"dense_{name}_w"], golden[f"dense_{name}_ids"]
    ref = golden[f"dense_{name}_scores"]
    tol = 1e-6 * np.linalg.norm(w) * float(np.max(np.linalg.norm(x, axis=1)))
    repo = otf.Repository.dense(otf.FeatureStore(x, ids=ids))
    s = repo.score(w)
    assert s.dtype == np.float32
    assert np.max(np.abs(s.astype(np.float64) - ref)) <= tol
    # 4-term float32 chains accumulated in float64: within the documented error bound
    ex = exact_dense(x, w)
    assert np.all(np.abs(s - ex) <= dense_error_bound(s, x, w))
    np.testing.assert_array_equal(otf.score_dense(w, x), s)
    ranked = repo.rank(otf.LinearModel(w, 1, 4), 50, produced_at=2.5)
    assert ranked.model_version == 4 and ranked.produced_at == 2.5
    o_ids, o_sc, _ = O.top_k(s, 50, ids)
    np.testing.assert_array_equal(ranked.ids, o_ids)
    np.testing.assert_array_equal(ranked.scores, o_sc)
    assert ranked.scores.dtype == np.float64 and ranked.ids.dtype == np.int64
    ref_of = dict(zip(map(int, ids), ref.astype(np.float64)))
    assert_rank_parity(ranked.ids, golden[f"dense_{name}_rank_ids"], ref_of, tol)


def test_dense_edge_cases(otf):
    rng = np.random.default_rng(1)
    store = otf.FeatureStore(rng.standard_normal((10, 4)).astype(np.float32))
    np.testing.assert_array_equal(otf.score_dense(np.zeros(4), store), 0.0)
    assert not np.any(np.signbit(otf.score_dense(np.zeros(4), store)))
    data = rng.standard_normal((20, 6)).astype(np.float32)
    w = np.zeros(6)
    w[3] = 1.0
    np.testing.assert_array_equal(otf.score_dense(w, data), data[:, 3])
    with pytest.raises(otf.ConfigError):
        otf.score_dense(np.zeros(5), np.ones((2, 4), np.float32))
    repo = otf.Repository.dense(otf.FeatureStore(rng.standard_normal((37, 128)).astype(np.float32)))
    with pytest.raises(otf.ConfigError):
        repo.score(np.zeros(127))
    # w = 0: every score ties, the lowest ids win (tests/test_ranker.py:146-148)
    r = repo.rank(otf.LinearModel(np.zeros(128), 1), 7)
    assert list(r.ids) == list(range(7))
    assert len(repo.rank(otf.LinearModel(np.ones(128), 1), 0)) == 0
    w = rng.standard_normal(128)
    full = repo.rank(otf.LinearModel(w, 1), 1000)  # k >= N: full sort
    assert len(full) == 37
    assert list(full.ids) == O.full_sort_ids(repo.score(w), np.arange(37), 37)


@pytest.mark.parametrize("n,d", [(1, 128), (31, 128), (33, 256), (1000, 384), (517, 2048), (300, 4096), (77, 3)])
def test_dense_shapes_position_independent(otf, n, d):
    """Every row's score is the same whatever its position (exclusion == rebuild, shard-invariance)."""
    rng = np.random.default_rng(n + d)
    x = rng.standard_normal((n, d)).astype(np.float32)
    w = rng.standard_normal(d)
    s = otf.score_dense(w, x)
    perm = rng.permutation(n)
    np.testing.assert_array_equal(otf.score_dense(w, x[perm]), s[perm])
    ex = exact_dense(x, w)
    assert np.all(np.abs(s - ex) <= dense_error_bound(s, x, w))


def test_exclusion_equals_rebuild(otf):
    """tests/test_ranker.py:253-266: without_ids ranks exactly like a rebuilt store."""
    rng = np.random.default_rng(21)
    data = rng.standard_normal((200, 16)).astype(np.float32)
    names = [f"item-{i}" for i in range(200)]
    store = otf.FeatureStore(data, names=names)
    model = otf.LinearModel(rng.standard_normal(16), iteration=5, version=1)
    excluded = {int(i) for i in rng.choice(200, size=40, replace=False)}
    a = otf.Repository.dense(store).without_ids(excluded).rank(model, 25)
    keep = [i for i in range(200) if i not in excluded]
    b = otf.Repository.dense(store.subset(np.array(keep))).rank(model, 25)
    assert list(a.ids) == list(b.ids)
    np.testing.assert_array_equal(a.scores, b.scores)
    assert a.names == b.names
    r = otf.Repository.dense(store).without_ids({0, 1, 2})
    assert r.count == 197 and int(r.ids.min()) == 3


def test_repository_views(otf):
    rng = np.random.default_rng(3)
    x = rng.standard_normal((120, 16)).astype(np.float32)
    repo = otf.Repository.dense(otf.FeatureStore(x))
    assert repo.payload_bytes() == 120 * 16 * 4 and repo.count == 120 and repo.model_dim == 16
    vecs = rng.standard_normal((3, 16)).astype(np.float32)
    np.testing.assert_array_equal(repo.adapt_training_vectors(vecs), vecs)
    w = rng.standard_normal(16)
    b = repo.rank(otf.LinearModel(w, 1), 10)
    c = repo.rank(w, 10)  # a bare array is accepted as the model (ranker.py:59-60)
    assert list(b.ids) == list(c.ids)  # repeated calls are bitwise identical
    np.testing.assert_array_equal(b.scores, c.scores)


# ---------------------------------------------------------------------------------------------
# top_k (ranker.py:97-143)


def test_top_k_known_answers(otf, golden):
    r = otf.top_k(np.array([0.5, 2.0, -1.0, 2.0]), 10)
    assert list(r.ids) == [1, 3, 0, 2]
    np.testing.assert_array_equal(r.scores, [2.0, 2.0, 0.5, -1.0])
    assert list(otf.top_k(np.ones(10), 4).ids) == [0, 1, 2, 3]
    r = otf.top_k(golden["topk_ties_scores"], 100, ids=golden["topk_ties_ids_in"])
    np.testing.assert_array_equal(r.ids, golden["topk_ties_ids"])
    np.testing.assert_array_equal(r.scores, golden["topk_ties_out_scores"])
    np.testing.assert_array_equal(otf.top_k(golden["topk_rand_scores"], 50).ids, golden["topk_rand_ids"])
    np.testing.assert_array_equal(otf.top_k(golden["topk_signed_zero_scores"], 4).ids, golden["topk_signed_zero_ids"])
    np.testing.assert_array_equal(otf.top_k(golden["topk_f64_scores"], 1000).ids, golden["topk_f64_ids"])
    np.testing.assert_array_equal(otf.top_k(golden["topk_f64_scores"][:700], 5000).ids, golden["topk_full_ids"])
    r = otf.top_k(np.array([1.0, 3.0, 2.0]), 2, ids=np.array([7, 8, 9]), names=["a", "b", "c"])
    assert list(r.ids) == [8, 9] and r.names == ("b", "c")
    assert len(otf.top_k(np.ones(5), 0)) == 0
    with pytest.raises(otf.ConfigError):
        otf.top_k(np.ones(5), 2, ids=np.arange(4))


@pytest.mark.parametrize("n,k,dtype,kind", [
    (1, 1, np.float32, "rand"), (5000, 4999, np.float32, "rand"), (100_000, 1000, np.float32, "rand"),
    (100_000, 1000, np.float64, "rand"), (70_000, 5000, np.float32, "ties"), (50_000, 1000, np.float64, "ties"),
    (20_000, 20_000, np.float32, "rand"), (9000, 4097, np.float64, "rand"), (3000, 1000, np.float32, "equal"),
    (65_536, 300, np.float32, "neg"),
])
def test_top_k_matches_oracle(otf, n, k, dtype, kind):
    rng = np.random.default_rng(n + k)
    if kind == "rand":
        s = rng.standard_normal(n).astype(dtype)
    elif kind == "ties":
        s = rng.integers(-4, 5, size=n).astype(dtype)
    elif kind == "equal":
        s = np.full(n, 0.25, dtype=dtype)
    else:
        s = -np.abs(rng.standard_normal(n)).astype(dtype)
    ids = rng.permutation(n * 3)[:n].astype(np.int64)
    r = otf.top_k(s, k, ids=ids)
    o_ids, o_sc, _ = O.top_k(s, k, ids)
    np.testing.assert_array_equal(r.ids, o_ids)
    np.testing.assert_array_equal(r.scores, o_sc)


@pytest.mark.parametrize("n,k", [(5000, 700), (200_000, 1000), (20_000, 9000)])
def test_top_k_signed_ids(otf, n, k):
    """The reference accepts any int64 ids for top_k and Repository.quantized / binary; ties break
    toward the smallest SIGNED id (np.lexsort), so negative ids come first."""
    rng = np.random.default_rng(n + 3)
    s = rng.integers(-3, 4, size=n).astype(np.float32)  # heavy ties: the id order decides
    ids = rng.permutation(np.arange(-n, 2 * n, dtype=np.int64))[:n]
    ids[:3] = [np.iinfo(np.int64).min, np.iinfo(np.int64).max, -1]
    r = otf.top_k(s, k, ids=ids)
    o_ids, o_sc, _ = O.top_k(s, k, ids)
    np.testing.assert_array_equal(r.ids, o_ids)
    np.testing.assert_array_equal(r.scores, o_sc)
    cents = rng.standard_normal((4, 16, 2)).astype(np.float32)
    codes = rng.integers(0, 16, (n, 4), dtype=np.uint8)
    w = rng.standard_normal(8)
    pq = otf.Repository.quantized(otf.PQCodebook(cents), codes, ids=ids)
    o_ids, o_sc, _ = O.top_k(O.score_pq(w, cents, codes), k, ids)
    got = pq.rank(otf.LinearModel(w, 1, 1), k)
    np.testing.assert_array_equal(got.ids, o_ids)
    np.testing.assert_array_equal(got.scores, o_sc)


def test_top_k_affine_invariance(otf):
    rng = np.random.default_rng(5)
    for _ in range(20):
        s = rng.integers(0, 20, size=200).astype(np.float64)
        scale, shift = rng.uniform(0.25, 8.0), rng.uniform(-5, 5)
        assert list(otf.top_k(s, 25).ids) == list(otf.top_k(s * scale + shift, 25).ids)


# ---------------------------------------------------------------------------------------------
# PQ (pq.py:248-276) — bit-exact


@pytest.mark.parametrize("name", PQ)
def test_pq_bit_exact(otf, golden, name):
    cents, codes, w = golden[f"pq_{name}_cents"], golden[f"pq_{name}_codes"], golden[f"pq_{name}_w"]
    book = otf.PQCodebook(cents)
    lut = otf.build_score_lut(w, book)
    assert lut.tobytes() == golden[f"pq_{name}_lut"].tobytes()
    s = otf.score_codes(golden[f"pq_{name}_lut"], codes)
    assert s.tobytes() == golden[f"pq_{name}_scores"].tobytes()
    np.testing.assert_array_equal(otf.score_pq(w, book, codes), s)
    repo = otf.Repository.quantized(book, codes)
    assert repo.score(w).tobytes() == golden[f"pq_{name}_scores"].tobytes()
    r = repo.rank(otf.LinearModel(w, 1, 1), 40)
    np.testing.assert_array_equal(r.ids, golden[f"pq_{name}_rank_ids"])
    assert r.scores.tobytes() == golden[f"pq_{name}_rank_scores"].tobytes()
    assert repo.payload_bytes() == codes.size and repo.model_dim == w.size


@pytest.mark.parametrize("kind", ["edges", "ties", "tiny", "mixed", "huge"])
def test_pq_rank_screening_paths(otf, kind):
    """The M=16 rank scan screens in float32 and rescoring in float64 only where the float32
    interval straddles a bin edge (otf_pq.cu pq_scan16_f32bins). Force that path: LUT entries
    that are small dyadic numbers put every score exactly on a bin edge; heavy ties; tiny
    (float32-subnormal) entries; a mixture of magnitudes. Ranked ids/scores must equal the
    oracle's top_k of the reference float64 scores bit for bit."""
    rng = np.random.default_rng({"edges": 1, "ties": 2, "tiny": 3, "mixed": 4, "huge": 5}[kind])
    n, k = 30_000, 500
    if kind == "edges":
        cents = (rng.integers(-8, 9, (16, 256, 8)) / 8.0).astype(np.float32)
        w = np.zeros(128)
        w[::8] = 1.0  # LUT[m][j] = c[m, j, 0]: multiples of 1/8, sums land on bin edges
    elif kind == "ties":
        cents = np.repeat(rng.standard_normal((16, 4, 8)), 64, axis=1).astype(np.float32)
        w = rng.standard_normal(128)
    elif kind == "tiny":
        cents = (rng.standard_normal((16, 256, 8)) * 1e-30).astype(np.float32)
        w = rng.standard_normal(128) * 1e-15
    elif kind == "mixed":
        cents = (rng.standard_normal((16, 256, 8)) * 10.0 ** rng.integers(-6, 6, (16, 1, 1))).astype(np.float32)
        w = rng.standard_normal(128)
    else:  # LUT entries near the float32 range: partial float32 sums could overflow
        cents = (rng.standard_normal((16, 256, 8)) * 1e37).astype(np.float32)
        w = rng.standard_normal(128) * 10.0
    codes = rng.integers(0, 256, (n, 16), dtype=np.uint8)
    ref = O.score_pq(w, cents, codes)
    repo = otf.Repository.quantized(otf.PQCodebook(cents), codes)
    assert repo.score(w).tobytes() == ref.tobytes()
    r = repo.rank(otf.LinearModel(w, 1, 1), k)
    o_ids, o_sc, _ = O.top_k(ref, k)
    np.testing.assert_array_equal(r.ids, o_ids)
    assert r.scores.tobytes() == np.asarray(o_sc, np.float64).tobytes()


def test_pq_errors(otf):
    cents = np.random.default_rng(0).standard_normal((4, 8, 2)).astype(np.float32)
    book = otf.PQCodebook(cents)
    with pytest.raises(otf.ConfigError):
        otf.build_score_lut(np.zeros(7), book)
    with pytest.raises(otf.ConfigError):
        otf.Repository.quantized(book, np.zeros((3, 5), np.uint8))
    with pytest.raises(otf.CorruptionError):
        otf.Repository.quantized(book, np.full((3, 4), 9, np.uint8))
    lut = otf.build_score_lut(np.zeros(8), book)
    assert lut.shape == (4, 8) and not np.any(lut)


def test_pq_single_code_and_width_check(otf):
    rng = np.random.default_rng(2)
    lut = rng.standard_normal((16, 256))
    codes = rng.integers(0, 256, (5, 16)).astype(np.uint8)
    assert otf.score_codes(lut, codes[0]) == O.score_codes(lut, codes[:1])[0]
    with pytest.raises(otf.ConfigError):
        otf.score_codes(lut, codes[:, :15])


# ---------------------------------------------------------------------------------------------
# binary (ranker.py:78-94, binary.py:86-128)


@pytest.mark.parametrize("name", BIN)
def test_binary_parity(otf, golden, name):
    bits = int(name[1:])
    codes, w = golden[f"bin_{name}_codes"], golden[f"bin_{name}_w"]
    ref = golden[f"bin_{name}_scores"].astype(np.float64)
    tol = 1e-6 * np.linalg.norm(w) * np.sqrt(bits)
    s = otf.score_binary(w, codes, bits)
    assert s.dtype == np.float32
    assert np.max(np.abs(s - ref)) <= tol
    bits_f = O.unpack_bits(codes, bits).astype(np.float64)
    exact = bits_f @ w.astype(np.float32).astype(np.float64)
    # byte tables in float32 + 4-term float32 lane sums, summed in float64 (otf_binary.cu)
    mag = bits_f @ np.abs(w.astype(np.float32).astype(np.float64))
    assert np.all(np.abs(s - exact) <= np.spacing(np.abs(s)) * 0.5 + 2.0 ** -21 * mag + 1e-30)
    np.testing.assert_array_equal(otf.unpack_bits(codes[:20], bits), golden[f"bin_{name}_unpacked"])
    np.testing.assert_array_equal(otf.hamming_distance(codes, golden[f"bin_{name}_other"]), golden[f"bin_{name}_hamming"])
    frame = golden.get(f"bin_{name}_frame")
    m = frame.shape[1] if frame is not None else 128
    codec = otf.BinaryCodec(otf.TightFrame(frame if frame is not None else np.eye(bits, m)), np.zeros(m, np.float32)
                            if frame is None else golden[f"bin_{name}_center"])
    repo = otf.Repository.binary(codec, codes)
    np.testing.assert_array_equal(repo.score(w), s)
    r = repo.rank(otf.LinearModel(w, 1, 2), 30)
    o_ids, o_sc, _ = O.top_k(s, 30)
    np.testing.assert_array_equal(r.ids, o_ids)
    assert_rank_parity(r.ids, golden[f"bin_{name}_rank_ids"], dict(enumerate(ref)), tol)
    if frame is not None:
        got = otf.binarize(codec, golden[f"bin_{name}_vecs"])
        np.testing.assert_array_equal(got, codes)
        np.testing.assert_array_equal(repo.adapt_training_vectors(golden[f"bin_{name}_vecs"][:10]),
                                      golden[f"bin_{name}_adapted"])


def test_binary_edge_cases(otf):
    w = np.random.default_rng(0).standard_normal(32)
    np.testing.assert_array_equal(otf.score_binary(w, np.zeros((6, 4), np.uint8), 32), 0.0)
    np.testing.assert_allclose(otf.score_binary(w, np.full((3, 4), 0xFF, np.uint8), 32), w.sum(), rtol=1e-5)
    with pytest.raises(otf.ConfigError):
        otf.score_binary(np.zeros(16), np.zeros((2, 4), np.uint8), 32)
    packed = np.array([[0b00000001, 0b00000001]], dtype=np.uint8)
    bits = otf.unpack_bits(packed, 9)
    expected = np.zeros(9, np.float32)
    expected[0] = expected[8] = 1.0
    np.testing.assert_array_equal(bits[0], expected)
    # padding bits are ignored when scoring (count=output_bits)
    w13 = np.random.default_rng(1).standard_normal(13)
    a = otf.score_binary(w13, np.array([[0xFF, 0x1F]], np.uint8), 13)
    b = otf.score_binary(w13, np.array([[0xFF, 0xFF]], np.uint8), 13)
    np.testing.assert_array_equal(a, b)


# ---------------------------------------------------------------------------------------------
# Pegasos (trainer.py:51-173)


def test_pegasos_known_answers(otf):
    cfg = otf.TrainerConfig(lam=1.0, batch_size=2, seed=0)
    w1 = otf.pegasos_step(np.zeros(2), 1, np.array([[1.0, 0.0]]), np.array([[0.0, 1.0]]), cfg, np.random.default_rng(0))
    np.testing.assert_allclose(w1, [0.5, -0.5], rtol=1e-12)
    w5 = otf.pegasos_step(np.array([2.0, 0.0]), 5, np.array([[1.1, 0.0]]), np.array([[-1.1, 0.0]]),
                          otf.TrainerConfig(lam=0.04, batch_size=2), np.random.default_rng(0))
    np.testing.assert_allclose(w5, [1.6, 0.0], rtol=1e-12)
    w2 = otf.pegasos_step(np.array([1.0, 0.0]), 2, np.array([[0.5, 0.0]]), np.array([[-3.0, 0.0]]),
                          otf.TrainerConfig(lam=0.25, batch_size=2), np.random.default_rng(0))
    np.testing.assert_allclose(w2, [1.0, 0.0], rtol=1e-12)
    capped = otf.pegasos_step(np.zeros(2), 1, np.array([[1.0, 0.0]]), np.array([[-1.0, 0.0]]),
                              otf.TrainerConfig(lam=0.01, batch_size=2), np.random.default_rng(0))
    np.testing.assert_allclose(np.linalg.norm(capped), 10.0, rtol=1e-12)
    free = otf.pegasos_step(np.zeros(2), 1, np.array([[1.0, 0.0]]), np.array([[-1.0, 0.0]]),
                            otf.TrainerConfig(lam=0.01, batch_size=2, project=False), np.random.default_rng(0))
    np.testing.assert_allclose(np.linalg.norm(free), 100.0, rtol=1e-12)
    with pytest.raises(otf.NotReadyError):
        otf.pegasos_step(np.zeros(2), 1, np.empty((0, 2)), np.ones((1, 2)), cfg, np.random.default_rng(0))
    with pytest.raises(otf.InsufficientDataError):
        otf.pegasos_step(np.zeros(2), 1, np.ones((1, 2)), np.empty((0, 2)), cfg, np.random.default_rng(0))


def test_pegasos_sequence_matches_reference(otf, golden):
    pos, neg = golden["peg_pos"], golden["peg_neg"]
    rng = np.random.default_rng(5)
    w = np.zeros(pos.shape[1])
    cfg = otf.TrainerConfig(lam=0.3, batch_size=8, project=False, seed=0)
    for t in range(1, 31):
        w = otf.pegasos_step(w, t, pos.astype(np.float64), neg.astype(np.float64), cfg, rng)
        np.testing.assert_allclose(w, golden["peg_noproj_w"][t - 1], rtol=1e-12, atol=1e-15)


def test_online_trainer_matches_reference(otf, golden):
    pos, neg = golden["peg_pos"], golden["peg_neg"]
    idx = []
    tr = otf.OnlineTrainer(pos.shape[1], neg, otf.TrainerConfig(lam=0.05, batch_size=16, seed=9),
                           batch_hook=lambda p, q: idx.append(np.concatenate([p, q])))
    with pytest.raises(otf.NotReadyError):
        tr.snapshot()
    for t in range(60):
        assert tr.step(pos) == t + 1
        snap = tr.snapshot()
        np.testing.assert_allclose(snap.weights, golden["peg_w"][t], rtol=1e-12, atol=1e-15)
        assert snap.iteration == t + 1 and snap.version == t + 1
    np.testing.assert_array_equal(np.stack(idx), golden["peg_idx"])
    again = tr.snapshot()
    assert again.version == 60
    with pytest.raises(ValueError):
        again.weights[0] = 1.0


def test_online_trainer_float64_negatives_are_stored_float32(otf, golden):
    """trainer.py:127: OnlineTrainer keeps np.asarray(negatives, dtype=np.float32) whatever the
    input dtype; pegasos_step then widens those float32 rows. float64 negatives that are not
    float32-representable must follow the same trajectory as the reference (not their exact
    float64 values)."""
    import otf_oracle as O

    pos, neg = golden["peg_pos"], golden["peg_neg"]
    neg64 = neg.astype(np.float64) + np.random.default_rng(3).standard_normal(neg.shape) * 1e-5
    assert not np.array_equal(neg64.astype(np.float32).astype(np.float64), neg64)
    cfg = otf.TrainerConfig(lam=0.05, batch_size=16, seed=9)
    tr = otf.OnlineTrainer(pos.shape[1], neg64, cfg)
    rng = np.random.default_rng(9)
    w = np.zeros(pos.shape[1])
    neg_ref = neg64.astype(np.float32).astype(np.float64)
    for t in range(1, 31):
        tr.step(pos)
        w = O.pegasos_step(w, t, pos.astype(np.float64), neg_ref, cfg.lam, cfg.batch_size, cfg.project, rng)
        np.testing.assert_allclose(tr.snapshot().weights, w, rtol=1e-12, atol=1e-15)


def test_online_trainer_device_pool_equals_host_pool(otf, golden):
    pos, neg = golden["peg_pos"], golden["peg_neg"]
    a = otf.OnlineTrainer(pos.shape[1], neg, otf.TrainerConfig(lam=0.05, batch_size=16, seed=9))
    b = otf.OnlineTrainer(pos.shape[1], neg, otf.TrainerConfig(lam=0.05, batch_size=16, seed=9))
    b.append_positives(pos[:10])
    assert b.append_positives(pos[10:]) == len(pos)
    for _ in range(40):
        a.step(pos)
        b.step()
    np.testing.assert_array_equal(a.snapshot().weights, b.snapshot().weights)


# ---------------------------------------------------------------------------------------------
# fixed-set SVM (trainer.py:197-257)


@pytest.mark.parametrize("name,epochs,seed", [("tb16", 20, 41), ("tb128", 8, 42)])
def test_train_batch_matches_reference(otf, golden, name, epochs, seed):
    pos, neg = golden[f"tb_{name}_pos"], golden[f"tb_{name}_neg"]
    hist = []
    model = otf.train_batch(pos, neg, otf.BatchTrainConfig(c=0.25, epochs=epochs, seed=seed), objective_history=hist)
    assert model.iteration == int(golden[f"tb_{name}_iter"][0])
    np.testing.assert_allclose(model.weights, golden[f"tb_{name}_w"], rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(np.array(hist), golden[f"tb_{name}_hist"], rtol=1e-10)
    feats = np.concatenate([pos, neg]).astype(np.float64)
    labels = np.concatenate([np.ones(len(pos)), -np.ones(len(neg))])
    lam = 1.0 / (0.25 * len(feats))
    np.testing.assert_allclose(otf.hinge_objective(model.weights, feats, labels, lam), golden[f"tb_{name}_obj"][0],
                               rtol=1e-9)


def test_train_batch_reference_behaviour(otf):
    """tests/test_trainer.py:245-306 of the reference, on the GPU trainer."""
    pos = np.array([[1.0, 0.0, 0.0, 0.0]])
    neg = np.array([[-1.0, 0.0, 0.0, 0.0]])
    m = otf.train_batch(pos, neg, otf.BatchTrainConfig(epochs=200, seed=0))
    assert m.weights[0] / np.linalg.norm(m.weights) > 0.999
    np.testing.assert_allclose(m.weights[0], 0.5, atol=0.05)
    rng = np.random.default_rng(19)
    p4 = O.normalize_rows(rng.standard_normal((8, 4)) + 1)
    n4 = O.normalize_rows(rng.standard_normal((8, 4)) - 1)
    assert otf.train_batch(p4, n4, otf.BatchTrainConfig(batch_size=4, epochs=5, seed=0)).iteration == 20
    a = otf.train_batch(p4, n4, otf.BatchTrainConfig(epochs=30, seed=7))
    b = otf.train_batch(p4, n4, otf.BatchTrainConfig(epochs=30, seed=7))
    assert a.weights.tobytes() == b.weights.tobytes()
    with pytest.raises(otf.InsufficientDataError):
        otf.train_batch(np.empty((0, 4)), np.ones((3, 4)))
    with pytest.raises(otf.ConfigError):
        otf.BatchTrainConfig(c=0.0).validate()


# ---- pq_encode (pq.py:206-230), the PQ ingest path ----------------------------------------------
def _codes_agree(gpu, ref, gap, cents, vecs):
    """Codes equal the reference's except at genuine near-ties: where they differ, the two
    centroids' float64 distances must agree to rounding level (BLAS dot order)."""
    bad = np.argwhere(gpu != ref)
    for i, m in bad:
        q = cents.shape[2]
        x = vecs[i, m * q:(m + 1) * q].astype(np.float64)
        c = cents[m].astype(np.float64)
        d = (c * c).sum(1) - 2.0 * (c @ x)
        a, b = d[int(gpu[i, m])], d[int(ref[i, m])]
        assert abs(a - b) <= 1e-12 * max(1.0, abs(a), abs(b)), (i, m, a, b)
    return len(bad)


@pytest.mark.parametrize("name", ["e16", "e4k16"])
def test_pq_encode_matches_reference_golden(otf, golden, name):
    cents, vecs = golden[f"pqenc_{name}_cents"], golden[f"pqenc_{name}_vecs"]
    book = otf.PQCodebook(cents)
    codes = otf.pq_encode(book, vecs)
    assert codes.dtype == np.uint8 and codes.shape == golden[f"pqenc_{name}_codes"].shape
    np.testing.assert_array_equal(codes, golden[f"pqenc_{name}_codes"])
    np.testing.assert_array_equal(otf.pq_encode(book, vecs[3]), golden[f"pqenc_{name}_codes"][3])  # single


@pytest.mark.parametrize("m,k,q,n", [(16, 256, 8, 20_000), (8, 256, 16, 5000), (3, 100, 7, 3000),
                                     (2, 256, 40, 1000), (32, 256, 4, 4000), (4, 100, 8, 3001), (5, 3, 8, 777)])
def test_pq_encode_matches_oracle(otf, m, k, q, n):
    rng = np.random.default_rng(m * 1000 + q)
    cents = rng.standard_normal((m, k, q)).astype(np.float32)
    cents[:, 1] = cents[:, 0]  # duplicate centroid: exact tie -> lowest index
    vecs = rng.standard_normal((n, m * q)).astype(np.float32)
    ref, gap = O.pq_encode(cents, vecs)
    gpu = otf.pq_encode(otf.PQCodebook(cents), vecs)
    assert _codes_agree(gpu, ref, gap, cents, vecs) <= max(1, n * m // 100_000)
    assert not np.any(gpu == 1)  # the duplicate of centroid 0 is never chosen


@pytest.mark.parametrize("scale", [1e-20, 1e-3, 1e15])
def test_pq_encode_magnitudes(otf, scale):
    """Q = 8 runs on the tensor cores (TF32 split dots, index-in-mantissa argmin); extreme but
    finite magnitudes must give the same codes as the float64 oracle."""
    rng = np.random.default_rng(int(np.log10(scale)) + 40)
    cents = (rng.standard_normal((4, 64, 8)) * scale).astype(np.float32)
    vecs = (rng.standard_normal((2000, 32)) * scale).astype(np.float32)
    ref, gap = O.pq_encode(cents, vecs)
    gpu = otf.pq_encode(otf.PQCodebook(cents), vecs)
    assert _codes_agree(gpu, ref, gap, cents, vecs) <= 1


def test_pq_encode_errors_and_empty(otf):
    book = otf.PQCodebook(np.zeros((2, 4, 3), np.float32))
    with pytest.raises(otf.ConfigError):
        otf.pq_encode(book, np.zeros((5, 7), np.float32))
    assert otf.pq_encode(book, np.zeros((0, 6), np.float32)).shape == (0, 2)


# ---- codebook learning (pq.py:116-203) -----------------------------------------------------------
@pytest.mark.parametrize("name,q,k,iters,seed", [("a", 8, 64, 10, 3), ("b", 3, 16, 25, 4)])
def test_learn_pq_codebook_matches_reference_golden(otf, golden, name, q, k, iters, seed):
    """GPU Lloyd steps (assignment, objective, means) + host re-seeding reproduce the reference's
    codebooks bit-for-bit and its objective histories to rounding (the BLAS dot order)."""
    book = otf.learn_pq_codebook(golden[f"km_{name}_train"],
                                 otf.PQConfig(subdim=q, num_centroids=k, iterations=iters, seed=seed))
    np.testing.assert_array_equal(book.centroids, golden[f"km_{name}_cents"])
    np.testing.assert_array_equal(book.centering, golden[f"km_{name}_centering"])
    assert [len(h) for h in book.objective_history] == list(golden[f"km_{name}_hist_len"])
    for m, h in enumerate(book.objective_history):
        np.testing.assert_allclose(h, golden[f"km_{name}_hist"][m][:len(h)], rtol=1e-12)


def test_lloyd_traces_match_reference(otf, golden):
    from paper_1407_4764_b200.pq import _lloyd

    c, h = _lloyd(np.array([[0.0], [1.0], [2.0], [3.0]]), 2, 10, np.random.default_rng(0),
                  init=np.array([[0.0], [1000.0]]))  # forced empty cluster (tests/test_pq.py:47-56)
    np.testing.assert_array_equal(c, golden["km_hand_cents"])
    np.testing.assert_array_equal(h, golden["km_hand_hist"])
    c, h = _lloyd(golden["km_empty_data"], 8, 15, np.random.default_rng(1), init=golden["km_empty_init"])
    np.testing.assert_array_equal(c, golden["km_empty_cents"])
    np.testing.assert_allclose(h, golden["km_empty_hist"], rtol=1e-12)
    c, h = _lloyd(golden["km_empty_data"], 8, 0, np.random.default_rng(1), init=golden["km_empty_init"])
    assert h == [] and np.array_equal(c, golden["km_empty_init"])


def test_learn_pq_codebook_errors(otf):
    with pytest.raises(otf.ConfigError):
        otf.learn_pq_codebook(np.ones((10, 10), np.float32), otf.PQConfig(subdim=4, num_centroids=2))
    with pytest.raises(otf.InsufficientDataError):
        otf.learn_pq_codebook(np.ones((3, 4), np.float32), otf.PQConfig(subdim=2, num_centroids=8))
    with pytest.raises(otf.InsufficientDataError):  # too few distinct sub-vectors
        otf.learn_pq_codebook(np.ones((20, 4), np.float32), otf.PQConfig(subdim=2, num_centroids=4))


@pytest.mark.parametrize("seed", range(24))
def test_top_k_randomised_against_oracle(otf, seed):
    """Randomised top_k cases (sizes, k around the candidate cap, dtypes, tie densities, signed
    zeros, shuffled / huge ids): ids and float64 scores must equal the oracle's."""
    rng = np.random.default_rng(1000 + seed)
    n = int(rng.choice([1, 7, 1000, 8191, 8193, 50_000, 300_000]))
    k = int(rng.choice([0, 1, 17, 1000, 8192, 8193, n, n + 5]))
    dtype = np.float32 if rng.random() < 0.6 else np.float64
    kind = rng.choice(["normal", "few", "ties", "zeros", "const"])
    if kind == "normal":
        s = rng.standard_normal(n)
    elif kind == "few":
        s = rng.integers(-3, 4, n) / 7.0
    elif kind == "ties":
        s = np.round(rng.standard_normal(n) * 20) / 20
    elif kind == "zeros":
        s = np.where(rng.random(n) < 0.5, 0.0, -0.0) * (rng.random(n) < 0.9) + (rng.random(n) < 0.1) * rng.standard_normal(n)
    else:
        s = np.full(n, 1.25)
    s = s.astype(dtype)
    ids = None
    if rng.random() < 0.5:
        ids = rng.permutation(n).astype(np.int64) * int(rng.choice([1, 3, 1 << 40])) + int(rng.integers(0, 1000))
    r = otf.top_k(s, k, ids=ids)
    o_ids, o_sc, _ = O.top_k(s, k, ids)
    np.testing.assert_array_equal(r.ids, o_ids)
    np.testing.assert_array_equal(r.scores, o_sc)
