"""Repository files straight into HBM (§8 f3; csrc/otf_ingest.cu): Repository.load_features /
load_quantized / load_binary against the reference's loaders (store.py:139-163, pq.py:318-330,
binary.py:176-187) — the byte layouts of formats.py, the same errors for bad magic, version,
truncation, trailing bytes, empty stores, zero rows, out-of-range codes and padding bits (ports
of pkg/tests/test_pq.py::TestCodesFile, test_binary.py::TestBinaryCodesFile and the
test_store.py load tests), and repositories that score and rank bit-identically to the ones
built from the reference's in-memory arrays."""

import struct

import numpy as np
import pytest

import otf_oracle as O

pytestmark = pytest.mark.gpu


def head(magic, *fields, version=1):
    out = magic + struct.pack("<I", version)
    for fmt, v in fields:
        out += struct.pack(fmt, v)
    return out


def write_otfr(path, x, version=1):  # store.py:166-175
    path.write_bytes(head(b"OTFR", ("<I", x.shape[1]), ("<Q", x.shape[0]), version=version) +
                     np.ascontiguousarray(x, "<f4").tobytes())


def write_otfc(path, codes):  # pq.py:307-315
    path.write_bytes(head(b"OTFC", ("<Q", codes.shape[0]), ("<I", codes.shape[1])) + codes.tobytes())


def write_otfh(path, codes, bits):  # binary.py:163-173
    path.write_bytes(head(b"OTFH", ("<Q", codes.shape[0]), ("<I", bits)) + codes.tobytes())


def test_codes_byte_layout_and_round_trip(otf, tmp_path):
    """test_pq.py::TestCodesFile (byte layout, round trip, size)."""
    codes = np.array([[1, 2], [3, 4]], dtype=np.uint8)
    path = tmp_path / "codes.otfc"
    write_otfc(path, codes)
    assert path.read_bytes() == b"OTFC" + struct.pack("<I", 1) + struct.pack("<Q", 2) + struct.pack("<I", 2) + bytes([1, 2, 3, 4])
    rng = np.random.default_rng(81)
    cents = rng.standard_normal((5, 16, 3)).astype(np.float32)
    codes = rng.integers(0, 16, size=(37, 5)).astype(np.uint8)
    write_otfc(path, codes)
    assert path.stat().st_size == 20 + 37 * 5
    book = otf.PQCodebook(cents)
    w = rng.standard_normal(15)
    a = otf.Repository.load_quantized(book, path)
    b = otf.Repository.quantized(book, codes)
    assert a.count == 37 and a.kind == "pq"
    assert a.score(w).tobytes() == b.score(w).tobytes() == O.score_pq(w, cents, codes).tobytes()
    np.testing.assert_array_equal(a.rank(otf.LinearModel(w, 1, 1), 10).ids, b.rank(otf.LinearModel(w, 1, 1), 10).ids)


def test_codes_errors(otf, tmp_path):
    rng = np.random.default_rng(1)
    book = otf.PQCodebook(rng.standard_normal((2, 4, 2)).astype(np.float32))
    path = tmp_path / "codes.otfc"
    write_otfc(path, np.array([[0, 7]], dtype=np.uint8))
    with pytest.raises(otf.CorruptionError):  # out of range for 4 centroids (pq.py:326-329)
        otf.Repository.load_quantized(book, path)
    book8 = otf.PQCodebook(rng.standard_normal((2, 8, 2)).astype(np.float32))
    assert otf.Repository.load_quantized(book8, path).count == 1
    write_otfc(path, np.ones((10, 2), dtype=np.uint8))
    path.write_bytes(path.read_bytes()[:-1])
    with pytest.raises(otf.CorruptionError, match="truncated"):
        otf.Repository.load_quantized(book, path)
    write_otfc(path, np.ones((10, 2), dtype=np.uint8))
    path.write_bytes(path.read_bytes() + b"\0")
    with pytest.raises(otf.CorruptionError, match="trailing"):
        otf.Repository.load_quantized(book, path)
    path.write_bytes(b"OTFX" + path.read_bytes()[4:])
    with pytest.raises(otf.FormatError):
        otf.Repository.load_quantized(book, path)
    write_otfc(path, np.ones((3, 5), dtype=np.uint8))
    with pytest.raises(otf.ConfigError):  # 5 blocks for a 2-block codebook (ranker.py:188-189)
        otf.Repository.load_quantized(book, path)
    write_otfc(path, np.ones((3, 2), dtype=np.uint8))
    with pytest.raises(otf.ConfigError):
        otf.Repository.load_quantized(book, path, ids=np.arange(4))
    with pytest.raises(FileNotFoundError):
        otf.Repository.load_quantized(book, tmp_path / "missing.otfc")
    path.write_bytes(head(b"OTFC", ("<Q", 1 << 62), ("<I", 2)) + bytes(8))  # a corrupt count
    with pytest.raises(otf.CorruptionError, match="truncated"):
        otf.Repository.load_quantized(book, path)
    path.write_bytes(head(b"OTFC", ("<Q", (1 << 64) - 1), ("<I", 8)))  # rows x width overflows
    with pytest.raises(otf.CorruptionError, match="truncated"):
        otf.Repository.load_quantized(book, path)


def test_binary_round_trip_and_errors(otf, tmp_path):
    """test_binary.py::TestBinaryCodesFile (round trip, size, padding, truncation)."""
    rng = np.random.default_rng(6)
    frame = otf.TightFrame(np.linalg.qr(rng.standard_normal((19, 8)))[0][:, :8])
    codec = otf.BinaryCodec(frame, np.zeros(8, np.float32))
    codes = otf.binarize(codec, rng.standard_normal((15, 8)))
    path = tmp_path / "codes.otfh"
    write_otfh(path, codes, 19)
    assert path.stat().st_size == 20 + 15 * 3
    w = rng.standard_normal(19)
    a = otf.Repository.load_binary(codec, path)
    b = otf.Repository.binary(codec, codes)
    assert a.count == 15 and a.model_dim == 19
    assert a.score(w).tobytes() == b.score(w).tobytes()
    path.write_bytes(head(b"OTFH", ("<Q", 1), ("<I", 13)) + bytes([0x00, 0xFF]))
    codec13 = otf.BinaryCodec(otf.TightFrame(np.linalg.qr(rng.standard_normal((13, 4)))[0][:, :4]),
                              np.zeros(4, np.float32))
    with pytest.raises(otf.CorruptionError, match="padding"):
        otf.Repository.load_binary(codec13, path)
    write_otfh(path, codes, 19)
    path.write_bytes(path.read_bytes()[:-2])
    with pytest.raises(otf.CorruptionError, match="truncated"):
        otf.Repository.load_binary(codec, path)
    write_otfh(path, codes, 19)
    with pytest.raises(otf.ConfigError):  # the codec's width (ranker.py:205-206)
        otf.Repository.load_binary(codec13, path)
    path.write_bytes(head(b"OTFH", ("<Q", 1), ("<I", 19), version=2) + bytes(3))
    with pytest.raises(otf.FormatError, match="version"):
        otf.Repository.load_binary(codec, path)


def test_features_normalised_bit_exact_and_names(otf, tmp_path):
    """load_features normalises on the device exactly as normalize_rows (store.py:32-53)."""
    rng = np.random.default_rng(3)
    for n, d in [(1, 3), (517, 128), (300, 200), (64, 2048), (9, 4096)]:
        x = (rng.standard_normal((n, d)) * rng.uniform(1e-3, 1e3, (n, 1))).astype(np.float32)
        path = tmp_path / "f.otfr"
        write_otfr(path, x)
        a = otf.Repository.load_features(path)
        b = otf.Repository.dense(O.normalize_rows(x))
        w = rng.standard_normal(d)
        assert a.count == n and a.model_dim == d and a.names is None
        assert a.score(w).tobytes() == b.score(w).tobytes()
        raw = otf.Repository.load_features(path, normalize=False)
        assert raw.score(w).tobytes() == otf.Repository.dense(x).score(w).tobytes()
    names = [f"img_{i:04d}.jpg" for i in range(n)]
    (tmp_path / "f.otfr.names").write_text("".join(f"{s}\n" for s in names), encoding="utf-8")
    assert otf.Repository.load_features(path).names == names
    (tmp_path / "f.otfr.names").write_text("a\nb\n", encoding="utf-8")
    with pytest.raises(otf.CorruptionError):
        otf.Repository.load_features(path)


def test_features_errors(otf, tmp_path):
    """test_store.py load tests: bad magic, truncation, empty store, zero rows."""
    path = tmp_path / "f.otfr"
    x = np.ones((4, 3), np.float32)
    write_otfr(path, x)
    path.write_bytes(b"JUNK" + path.read_bytes()[4:])
    with pytest.raises(otf.FormatError, match="bad magic"):
        otf.Repository.load_features(path)
    write_otfr(path, x)
    path.write_bytes(path.read_bytes()[:-4])
    with pytest.raises(otf.CorruptionError, match="truncated"):
        otf.Repository.load_features(path)
    path.write_bytes(b"OTFR" + struct.pack("<I", 1) + struct.pack("<I", 3))  # no count field
    with pytest.raises(otf.CorruptionError, match="truncated"):
        otf.Repository.load_features(path)
    write_otfr(path, np.zeros((0, 3), np.float32))
    with pytest.raises(otf.EmptyStoreError):
        otf.Repository.load_features(path)
    y = np.ones((5, 3), np.float32)
    y[3] = 0.0
    write_otfr(path, y)
    with pytest.raises(otf.DegenerateInputError, match="row 3"):
        otf.Repository.load_features(path)
    assert otf.Repository.load_features(path, normalize=False).count == 5


def test_large_codes_file_ranks_identically(otf, tmp_path):
    """A 20M x 16 OTFC file (320 MB, 20 chunks over 4 reader threads) loads into a repository that
    ranks bit-identically to Repository.quantized on the same codes (the PQ cut path)."""
    rng = np.random.default_rng(11)
    cents = rng.standard_normal((16, 256, 8)).astype(np.float32)
    codes = rng.integers(0, 256, (20_000_000, 16), dtype=np.uint8)
    path = tmp_path / "big.otfc"
    write_otfc(path, codes)
    book = otf.PQCodebook(cents)
    a = otf.Repository.load_quantized(book, path)
    w = rng.standard_normal(128)
    r = a.rank(otf.LinearModel(w, 1, 1), 1000)
    o_ids, o_sc, _ = O.top_k(O.score_pq(w, cents, codes), 1000)
    np.testing.assert_array_equal(r.ids, o_ids)
    assert r.scores.tobytes() == np.asarray(o_sc).tobytes()
