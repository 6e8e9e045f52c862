"""Multi-slice binary codes (2048 / 4096 / 8192 bits) on both scans: the per-slice launches (the
default) and the clustered one (bin_score_cluster: one CTA per 128-byte slice, the slice sums
meet over distributed shared memory). The scores must be
bit-identical to a numpy model of the kernel's fixed arithmetic (byte tables summed in float64
and rounded to float32, 4-term float32 lane sums, the float32 xor-tree over the 32 lanes, slices
chained in float64) and to the per-slice launches (the default; float64 partials through HBM), and within the
reference tolerance of the exact dot (ranker.py:78-94). The clustered kernel is opt-in
(OTF_BIN_CLUSTER=1, read per call): every case runs on both paths."""

import os
from pathlib import Path

import numpy as np
import pytest

import otf_oracle as O

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


def kernel_model(w, codes, n_bits):
    """float32 scores exactly as otf_binary.cu computes them (test infrastructure)."""
    n, rb = codes.shape
    w32 = np.zeros(rb * 8, np.float64)
    w32[:n_bits] = w.astype(np.float32).astype(np.float64)
    # T[p][v] = float32(sum, in bit order, of float32(w) over the set bits of v at byte position p)
    bits = ((np.arange(256)[:, None] >> np.arange(8)[None, :]) & 1).astype(bool)  # (256, 8)
    tab = np.zeros((rb, 256), np.float32)
    for p in range(rb):
        acc = np.zeros(256, np.float64)
        for b in range(8):
            acc = np.where(bits[:, b], acc + w32[8 * p + b], acc)
        tab[p] = acc.astype(np.float32)
    total = np.zeros(n, np.float64)
    for sl in range(rb // 128):
        # lane l: bytes 4l..4l+3 of the slice, summed left to right in float32
        look = tab[sl * 128 + np.arange(128)[None, :], codes[:, sl * 128:(sl + 1) * 128]]  # (n, 128)
        look = look.reshape(n, 32, 4)
        a = ((look[:, :, 0] + look[:, :, 1]) + look[:, :, 2]) + look[:, :, 3]  # float32
        for half in (16, 8, 4, 2, 1):  # the xor tree over the lanes (float32)
            a = a[:, :half] + a[:, half:2 * half]
        total = total + a[:, 0].astype(np.float64) if sl else a[:, 0].astype(np.float64)
    return total.astype(np.float32)


@pytest.fixture(params=["per_slice", "cluster"])
def path(request):
    old = os.environ.pop("OTF_BIN_CLUSTER", None)
    if request.param == "cluster":
        os.environ["OTF_BIN_CLUSTER"] = "1"
    yield request.param
    os.environ.pop("OTF_BIN_CLUSTER", None)
    if old is not None:
        os.environ["OTF_BIN_CLUSTER"] = old


@pytest.mark.parametrize("n_bits,n", [(2048, 1), (2048, 31), (2048, 5000), (2048, 300_001), (4096, 7777),
                                      (8192, 3001), (4000, 513)])
def test_slices_bit_exact(otf, path, n_bits, n):
    rng = np.random.default_rng(n_bits + n)
    rb = (n_bits + 7) // 8
    codes = rng.integers(0, 256, (n, rb), dtype=np.uint8)
    w = rng.standard_normal(n_bits)
    s = otf.score_binary(w, codes, n_bits)
    if n_bits % 1024 == 0:  # whole 128-byte slices: the byte-table kernels
        np.testing.assert_array_equal(s, kernel_model(w, codes, n_bits))
    ref = O.score_binary(w, codes, n_bits)
    tol = 1e-6 * np.linalg.norm(w) * np.sqrt(n_bits)
    assert np.max(np.abs(s.astype(np.float64) - ref)) <= tol
    ids, _, _ = O.top_k(s, min(n, 50))
    codec = otf.BinaryCodec(otf.TightFrame(np.eye(n_bits, 8)), np.zeros(8, np.float32))
    repo = otf.Repository.binary(codec, codes)
    np.testing.assert_array_equal(repo.rank(otf.LinearModel(w, 1, 1), min(n, 50)).ids, ids)


def test_cluster_equals_per_slice_launches(otf):
    rng = np.random.default_rng(5)
    codes = rng.integers(0, 256, (200_003, 256), dtype=np.uint8)
    w = rng.standard_normal(2048)
    os.environ.pop("OTF_BIN_CLUSTER", None)
    a = otf.score_binary(w, codes, 2048)
    os.environ["OTF_BIN_CLUSTER"] = "1"
    try:
        b = otf.score_binary(w, codes, 2048)
    finally:
        os.environ.pop("OTF_BIN_CLUSTER", None)
    assert a.tobytes() == b.tobytes()


def test_wide_equals_narrow_loads(otf, tmp_path):
    """The default binary scan (16-byte loads per lane, rotated virtual lanes) and the round-1 form
    (OTF_BIN_NARROW=1: one 4-byte load per lane and row; read once per process, so it runs in a
    subprocess) give the same bits for 2048- and 4096-bit codes with a ragged row count."""
    import subprocess
    import sys

    rng = np.random.default_rng(17)
    for n_bits, n in ((2048, 100_003), (4096, 33_333)):
        codes = rng.integers(0, 256, (n, n_bits // 8), dtype=np.uint8)
        w = rng.standard_normal(n_bits)
        np.save(tmp_path / "codes.npy", codes)
        np.save(tmp_path / "w.npy", w)
        wide = otf.score_binary(w, codes, n_bits)
        script = (
            "import sys, numpy as np; sys.path.insert(0, %r); import paper_1407_4764_b200 as otf; "
            "c = np.load(%r); w = np.load(%r); np.save(%r, otf.score_binary(w, c, %d))"
            % (str(ROOT), str(tmp_path / "codes.npy"), str(tmp_path / "w.npy"), str(tmp_path / "narrow.npy"), n_bits))
        env = dict(os.environ, OTF_BIN_NARROW="1")
        subprocess.run([sys.executable, "-c", script], check=True, env=env, timeout=600)
        narrow = np.load(tmp_path / "narrow.npy")
        assert wide.tobytes() == narrow.tobytes()


def test_adopted_codes_at_4_byte_offset(otf):
    """A borrowed device buffer whose rows start 4 bytes past a 16-byte boundary (allowed by the
    byte-table path) takes the narrow loads: same scores and ranking as an aligned copy."""
    import torch

    rng = np.random.default_rng(23)
    n, n_bits = 50_001, 2048
    codes = rng.integers(0, 256, (n, n_bits // 8), dtype=np.uint8)
    w = rng.standard_normal(n_bits)
    buf = torch.empty(codes.size + 16, dtype=torch.uint8, device="cuda")
    buf[4:4 + codes.size].copy_(torch.from_numpy(codes.reshape(-1)))
    off = otf.Repository.from_device("binary", buf.data_ptr() + 4, n, n_bits)
    ref = otf.score_binary(w, codes, n_bits)
    assert off.score(w).tobytes() == ref.tobytes()
    ids, _, _ = O.top_k(ref, 100)
    np.testing.assert_array_equal(off.rank(otf.LinearModel(w, 1, 1), 100).ids, ids)
    del off, buf
