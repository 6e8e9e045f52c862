"""Parity at BASELINE.json sizes (GPU box only; data generated on the device, checked on the host).

Size-independent properties at full scale:
  * C2 1M x 2048 dense: rank(k=1000) == the oracle's exact top_k of the GPU's own scores (selection
    is exact), the scores of a random row sample agree with a float64 host dot within the kernel
    bound, and rank is bitwise repeatable.
  * C3 10M PQ-16: every score and the top-1000 bit-identical to the numpy oracle (pq.py:248-276).
  * C5a binary 2048-bit (10M rows here): top-1000 == oracle top_k of the GPU scores; a row sample
    matches the exact bit-weight sum within the documented bound.
"""

import ctypes as C

import numpy as np
import pytest

import otf_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def test_c2_dense_1m_x_2048(otf, torch_cuda):
    torch = torch_cuda
    n, d, k = 1_000_000, 2048, 1000
    g = torch.Generator(device="cuda").manual_seed(7)
    x = torch.randn((n, d), device="cuda", generator=g)
    x /= x.norm(dim=1, keepdim=True)
    repo = otf.Repository.from_device("dense", x.data_ptr(), n, d)
    w = np.random.default_rng(3).standard_normal(d)
    s = repo.score(w)
    r1 = repo.rank(otf.LinearModel(w, 1, 1), k)
    r2 = repo.rank(otf.LinearModel(w, 1, 1), k)
    o_ids, o_sc, _ = O.top_k(s, k)
    np.testing.assert_array_equal(r1.ids, o_ids)
    np.testing.assert_array_equal(r1.scores, o_sc)
    assert r1.ids.tobytes() == r2.ids.tobytes() and r1.scores.tobytes() == r2.scores.tobytes()
    rows = np.random.default_rng(4).choice(n, 2000, replace=False)
    xs = x[torch.as_tensor(rows, device="cuda")].cpu().numpy()
    ex = xs.astype(np.float64) @ w.astype(np.float32).astype(np.float64)
    mag = np.abs(xs.astype(np.float64)) @ np.abs(w.astype(np.float32).astype(np.float64))
    assert np.all(np.abs(s[rows] - ex) <= np.spacing(np.abs(s[rows])) * 0.5 + 2.0 ** -22 * mag)
    # the top entries are the rows with the largest exact scores (tolerance only at near-ties)
    top = r1.ids[:50]
    xt = x[torch.as_tensor(top, device="cuda")].cpu().numpy().astype(np.float64)
    et = xt @ w.astype(np.float32).astype(np.float64)
    assert np.all(np.diff(et) <= 1e-6 * np.linalg.norm(w))


def test_c3_pq_10m_bit_exact(otf, torch_cuda):
    torch = torch_cuda
    n, m, q, k = 10_000_000, 16, 8, 1000
    g = torch.Generator(device="cuda").manual_seed(11)
    codes = torch.randint(0, 256, (n, m), dtype=torch.uint8, device="cuda", generator=g)
    cents = np.random.default_rng(12).standard_normal((m, 256, q)).astype(np.float32)
    w = np.random.default_rng(13).standard_normal(m * q)
    repo = otf.Repository.from_device("pq", codes.data_ptr(), n, m, codebook=otf.PQCodebook(cents))
    s = repo.score(w)
    host_codes = codes.cpu().numpy()
    ref = O.score_pq(w, cents, host_codes)
    assert s.tobytes() == ref.tobytes()
    r = repo.rank(otf.LinearModel(w, 1, 1), k)
    o_ids, o_sc, _ = O.top_k(ref, k)
    np.testing.assert_array_equal(r.ids, o_ids)
    assert r.scores.tobytes() == o_sc.tobytes()


def test_c5a_binary_10m(otf, torch_cuda):
    torch = torch_cuda
    n, bits, k = 10_000_000, 2048, 1000
    g = torch.Generator(device="cuda").manual_seed(21)
    codes = torch.empty((n, bits // 8), dtype=torch.uint8, device="cuda")
    codes.random_(0, 256, generator=g)
    repo = otf.Repository.from_device("binary", codes.data_ptr(), n, bits)
    w = np.random.default_rng(22).standard_normal(bits)
    s = repo.score(w)
    r = repo.rank(otf.LinearModel(w, 1, 1), k)
    o_ids, o_sc, _ = O.top_k(s, k)
    np.testing.assert_array_equal(r.ids, o_ids)
    rows = np.random.default_rng(23).choice(n, 500, replace=False)
    cs = codes[torch.as_tensor(rows, device="cuda")].cpu().numpy()
    bitsf = O.unpack_bits(cs, bits).astype(np.float64)
    w32 = w.astype(np.float32).astype(np.float64)
    ex = bitsf @ w32
    mag = bitsf @ np.abs(w32)
    assert np.all(np.abs(s[rows] - ex) <= np.spacing(np.abs(s[rows])) * 0.5 + 2.0 ** -21 * mag)
    ref = O.score_binary(w, cs, bits)  # the reference's own float32 sgemv path
    assert np.max(np.abs(s[rows].astype(np.float64) - ref)) <= 1e-6 * np.linalg.norm(w) * np.sqrt(bits)
