"""The CPU oracle (oracle/otf_oracle.py) pinned against the real reference's outputs.

tests/golden/golden.npz was produced by tests/golden/make_golden.py running the unmodified
reference (otf_retrieval) — these tests prove the oracle reproduces it, so the GPU parity tests
that compare against the oracle inherit the pin. CPU only.
"""

import numpy as np
import pytest

import otf_oracle as O

DENSE = ["d16", "d128", "d2048", "d5"]
PQ = ["m4k8q4", "m16k256q8", "m5k7q3", "m32k256q4", "m12k200q16", "m200k16q1"]
BIN = ["b32", "b2048", "b19", "b1024"]


@pytest.mark.parametrize("name", DENSE)
def test_dense_scores_and_rank(golden, name):
    x, w, ids = golden[f"dense_{name}_x"], golden[f"dense_{name}_w"], golden[f"dense_{name}_ids"]
    s = O.score_dense(w, x)
    np.testing.assert_array_equal(s, golden[f"dense_{name}_scores"])
    rid, rsc, _ = O.top_k(s, 50, ids)
    np.testing.assert_array_equal(rid, golden[f"dense_{name}_rank_ids"])
    np.testing.assert_array_equal(rsc, golden[f"dense_{name}_rank_scores"])


@pytest.mark.parametrize("name", PQ)
def test_pq_lut_and_scores_bit_exact(golden, name):
    cents, codes, w = golden[f"pq_{name}_cents"], golden[f"pq_{name}_codes"], golden[f"pq_{name}_w"]
    lut = O.build_score_lut(w, cents)
    assert lut.tobytes() == golden[f"pq_{name}_lut"].tobytes()
    s = O.score_codes(lut, codes)
    assert s.tobytes() == golden[f"pq_{name}_scores"].tobytes()
    rid, rsc, _ = O.top_k(s, 40)
    np.testing.assert_array_equal(rid, golden[f"pq_{name}_rank_ids"])
    assert rsc.tobytes() == golden[f"pq_{name}_rank_scores"].tobytes()


@pytest.mark.parametrize("name", PQ)
def test_explicit_orders_reproduce_reference_bits(golden, name):
    """The scalar orders the CUDA kernels implement equal the reference's numpy results."""
    cents, codes, w = golden[f"pq_{name}_cents"], golden[f"pq_{name}_codes"], golden[f"pq_{name}_w"]
    m, k, q = cents.shape
    ref_lut = golden[f"pq_{name}_lut"]
    wb = w.reshape(m, q)
    for mm in range(m):
        for j in range(0, k, max(1, k // 17)):
            assert O.lut_entry_numpy_order(cents[mm, j].astype(np.float64), wb[mm]) == ref_lut[mm, j]
    ref_s = golden[f"pq_{name}_scores"]
    for i in range(0, codes.shape[0], max(1, codes.shape[0] // 50)):
        vals = ref_lut[np.arange(m), codes[i]]
        assert O.pairwise_sum_numpy_order(list(vals)) == ref_s[i]


@pytest.mark.parametrize("q", list(range(1, 20)) + [32, 33, 64])
def test_einsum_order_probe_on_this_host(q):
    """numpy's einsum order is a property of the host numpy build: re-probe it wherever tests run."""
    rng = np.random.default_rng(q)
    c = (rng.standard_normal((3, 64, q)) * np.exp(rng.uniform(-8, 8, (3, 64, q)))).astype(np.float32)
    w = rng.standard_normal(3 * q) * np.exp(rng.uniform(-8, 8, 3 * q))
    lut = np.einsum("mkq,mq->mk", c.astype(np.float64), w.reshape(3, q))
    for m in range(3):
        for j in range(64):
            assert O.lut_entry_numpy_order(c[m, j].astype(np.float64), w.reshape(3, q)[m]) == lut[m, j]


@pytest.mark.parametrize("m", list(range(1, 40)) + [64, 127, 128, 129, 200, 256, 512])
def test_pairwise_order_probe_on_this_host(m):
    rng = np.random.default_rng(m)
    lut = rng.standard_normal((m, 256)) * np.exp(rng.uniform(-15, 15, (m, 1)))
    codes = rng.integers(0, 256, (40, m), dtype=np.uint8)
    got = lut[np.arange(m), codes].sum(axis=1)
    for i in range(40):
        assert O.pairwise_sum_numpy_order(list(lut[np.arange(m), codes[i]])) == got[i]


@pytest.mark.parametrize("name", BIN)
def test_binary_paths(golden, name):
    bits = int(name[1:])
    codes, w = golden[f"bin_{name}_codes"], golden[f"bin_{name}_w"]
    s = O.score_binary(w, codes, bits)
    np.testing.assert_array_equal(s, golden[f"bin_{name}_scores"])
    np.testing.assert_array_equal(O.unpack_bits(codes[:20], bits), golden[f"bin_{name}_unpacked"])
    np.testing.assert_array_equal(O.hamming_distance(codes, golden[f"bin_{name}_other"]), golden[f"bin_{name}_hamming"])
    rid, rsc, _ = O.top_k(s, 30)
    np.testing.assert_array_equal(rid, golden[f"bin_{name}_rank_ids"])
    if f"bin_{name}_frame" in golden:
        m = golden[f"bin_{name}_frame"].shape[1]
        frame = O.make_tight_frame(m, bits, seed={"b32": 21, "b19": 23, "b1024": 24}[name])
        assert frame.tobytes() == golden[f"bin_{name}_frame"].tobytes()
        got = O.binarize(frame, golden[f"bin_{name}_center"], golden[f"bin_{name}_vecs"])
        np.testing.assert_array_equal(got, codes)


def test_topk_known_answers(golden):
    ids, sc, _ = O.top_k(np.array([0.5, 2.0, -1.0, 2.0]), 10)
    assert list(ids) == [1, 3, 0, 2]
    assert list(sc) == [2.0, 2.0, 0.5, -1.0]
    assert list(O.top_k(np.ones(10), 4)[0]) == [0, 1, 2, 3]
    rid, _, _ = O.top_k(golden["topk_ties_scores"], 100, golden["topk_ties_ids_in"])
    np.testing.assert_array_equal(rid, golden["topk_ties_ids"])
    assert list(rid) == O.full_sort_ids(golden["topk_ties_scores"], golden["topk_ties_ids_in"], 100)
    np.testing.assert_array_equal(O.top_k(golden["topk_rand_scores"], 50)[0], golden["topk_rand_ids"])
    np.testing.assert_array_equal(O.top_k(golden["topk_signed_zero_scores"], 4)[0], golden["topk_signed_zero_ids"])
    np.testing.assert_array_equal(O.top_k(golden["topk_f64_scores"], 1000)[0], golden["topk_f64_ids"])
    np.testing.assert_array_equal(O.top_k(golden["topk_f64_scores"][:700], 5000)[0], golden["topk_full_ids"])
    assert len(O.top_k(np.ones(5), 0)[0]) == 0


def test_pegasos_known_answers():
    """tests/test_trainer.py:62-98 of the reference."""
    rng = np.random.default_rng(0)
    w1 = O.pegasos_step(np.zeros(2), 1, np.array([[1.0, 0.0]]), np.array([[0.0, 1.0]]), 1.0, 2, True, rng)
    np.testing.assert_allclose(w1, [0.5, -0.5], rtol=1e-12)
    w5 = O.pegasos_step(np.array([2.0, 0.0]), 5, np.array([[1.1, 0.0]]), np.array([[-1.1, 0.0]]), 0.04, 2, True,
                        np.random.default_rng(0))
    np.testing.assert_allclose(w5, [1.6, 0.0], rtol=1e-12)
    w2 = O.pegasos_step(np.array([1.0, 0.0]), 2, np.array([[0.5, 0.0]]), np.array([[-3.0, 0.0]]), 0.25, 2, True,
                        np.random.default_rng(0))
    np.testing.assert_allclose(w2, [1.0, 0.0], rtol=1e-12)


def test_pegasos_sequence_matches_reference(golden):
    pos, neg = golden["peg_pos"], golden["peg_neg"]
    rng = np.random.default_rng(9)
    w = np.zeros(pos.shape[1])
    idx = []
    for t in range(1, 61):
        w = O.pegasos_step(w, t, pos, neg, 0.05, 16, True, rng, hook=lambda p, q: idx.append(np.concatenate([p, q])))
        np.testing.assert_array_equal(w, golden["peg_w"][t - 1])
    np.testing.assert_array_equal(np.stack(idx), golden["peg_idx"])


@pytest.mark.parametrize("name,epochs,seed", [("tb16", 20, 41), ("tb128", 8, 42)])
def test_train_batch_matches_reference(golden, name, epochs, seed):
    pos, neg = golden[f"tb_{name}_pos"], golden[f"tb_{name}_neg"]
    hist = []
    w, total = O.train_batch(pos, neg, epochs=epochs, seed=seed, history=hist)
    np.testing.assert_array_equal(w, golden[f"tb_{name}_w"])
    assert total == int(golden[f"tb_{name}_iter"][0])
    np.testing.assert_array_equal(np.array(hist), golden[f"tb_{name}_hist"])


@pytest.mark.parametrize("name", ["e16", "e4k16"])
def test_oracle_pq_encode_matches_reference(golden, name):
    codes, gap = O.pq_encode(golden[f"pqenc_{name}_cents"], golden[f"pqenc_{name}_vecs"])
    np.testing.assert_array_equal(codes, golden[f"pqenc_{name}_codes"])
    assert np.all(gap >= 0)


@pytest.mark.parametrize("name,q,k,iters,seed", [("a", 8, 64, 10, 3), ("b", 3, 16, 25, 4)])
def test_oracle_learn_pq_codebook_matches_reference(golden, name, q, k, iters, seed):
    cents, hists, centering = O.learn_pq_codebook(golden[f"km_{name}_train"], q, k, iters, seed)
    np.testing.assert_array_equal(cents, golden[f"km_{name}_cents"])
    np.testing.assert_array_equal(centering, golden[f"km_{name}_centering"])
    for m, h in enumerate(hists):
        assert len(h) == golden[f"km_{name}_hist_len"][m]
        np.testing.assert_allclose(h, golden[f"km_{name}_hist"][m][:len(h)], rtol=1e-12)


def test_oracle_lloyd_traces(golden):
    c, h = O.lloyd(np.array([[0.0], [1.0], [2.0], [3.0]]), 2, 10, np.random.default_rng(0),
                   init=np.array([[0.0], [1000.0]]))
    np.testing.assert_array_equal(c, golden["km_hand_cents"])
    np.testing.assert_array_equal(h, golden["km_hand_hist"])
    c, h = O.lloyd(golden["km_empty_data"], 8, 15, np.random.default_rng(1), init=golden["km_empty_init"])
    np.testing.assert_array_equal(c, golden["km_empty_cents"])
    np.testing.assert_allclose(h, golden["km_empty_hist"], rtol=1e-12)
